// Read-bandwidth probe: which streaming-read pattern reaches the HBM read
// ceiling on B200?  Each kernel XOR-reduces a 1 GiB buffer (a result is
// written so nothing is dead code).
//   ld16   grid-stride, one 16-byte load per thread per iteration
//   ld64   four independent 16-byte loads per thread per iteration
//   bulk   per CTA a ring of shared-memory stages filled by cp.async.bulk
//          (TMA, mbarrier complete_tx), read back with LDS.128
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o read_probe read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ld16(const uint4 *p, size_t n, uint32_t *out)
{
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u)
        *out = acc;
}

__global__ void k_ld64(const uint4 *p, size_t n, uint32_t *out)
{
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i + 3 * stride < n; i += 4 * stride) {
        uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    if (acc == 0x12345678u)
        *out = acc;
}

template <int STAGES, int STAGE_BYTES>
__global__ void k_bulk(const uint8_t *p, size_t nbytes, uint32_t *out)
{
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    const size_t nchunks = nbytes / STAGE_BYTES;
    const uint32_t tid = threadIdx.x;
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](size_t c, int s) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm + s * STAGE_BYTES);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(STAGE_BYTES) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(p + c * STAGE_BYTES), "r"(STAGE_BYTES), "r"(b)
                     : "memory");
    };
    size_t c = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s)
            if (c + (size_t)s * gridDim.x < nchunks)
                issue(c + (size_t)s * gridDim.x, s);
    uint32_t acc = 0;
    uint32_t phase = 0;
    int s = 0;
    for (; c < nchunks; c += gridDim.x) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(b),
                     "r"(phase)
                     : "memory");
        const uint4 *v = reinterpret_cast<const uint4 *>(sm + s * STAGE_BYTES);
        for (int i = tid; i < STAGE_BYTES / 16; i += blockDim.x) {
            uint4 x = v[i];
            acc ^= x.x ^ x.y ^ x.z ^ x.w;
        }
        __syncthreads();
        if (tid == 0 && c + (size_t)STAGES * gridDim.x < nchunks)
            issue(c + (size_t)STAGES * gridDim.x, s);
        if (++s == STAGES) {
            s = 0;
            phase ^= 1;
        }
    }
    if (acc == 0x12345678u)
        *out = acc;
}

template <class F>
static float timeit(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i)
        f();
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i)
        f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main()
{
    const size_t nbytes = 1ull << 30;
    uint8_t *buf;
    uint32_t *out;
    cudaMalloc(&buf, nbytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, nbytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n16 = nbytes / 16;
    for (int per_sm : {4, 8}) {
        float ms = timeit([&] { k_ld16<<<sms * per_sm, 256>>>((const uint4 *)buf, n16, out); });
        printf("ld16 ctas/sm=%d: %.1f us  %.0f GB/s\n", per_sm, ms * 1e3, nbytes / ms / 1e6);
        ms = timeit([&] { k_ld64<<<sms * per_sm, 256>>>((const uint4 *)buf, n16, out); });
        printf("ld64 ctas/sm=%d: %.1f us  %.0f GB/s\n", per_sm, ms * 1e3, nbytes / ms / 1e6);
    }
#define BULK(ST, SB, CPS, THR)                                                                                         \
    {                                                                                                                  \
        auto k = k_bulk<ST, SB>;                                                                                       \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB);                                 \
        float ms = timeit([&] { k<<<sms * CPS, THR, ST * SB>>>(buf, nbytes, out); });                                  \
        printf("bulk stages=%d x %d B, ctas/sm=%d, thr=%d: %.1f us  %.0f GB/s  (%s)\n", ST, SB, CPS, THR, ms * 1e3,     \
               nbytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));                                             \
    }
    BULK(4, 16384, 1, 256)
    BULK(4, 16384, 2, 256)
    BULK(8, 8192, 2, 256)
    BULK(6, 16384, 2, 256)
    BULK(4, 32768, 1, 512)
    BULK(3, 32768, 2, 256)
    return 0;
}
