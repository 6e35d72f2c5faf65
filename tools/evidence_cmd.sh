# Round evidence: bench line, launch list (no extras), full ncu capture of K1-K4.
set -x
timeout -s USR1 -k 20 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_transcode|k_validate" --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_kernels.py --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_transcode|k_validate" -o gpurun_out/prof_${TAG:-r02} -f python tools/prof_kernels.py --reps 1 > gpurun_out/ncu_full.log 2>&1
echo rc=$?
