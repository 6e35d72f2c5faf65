"""Zero-copy smoke: K1 on pinned host buffers, small sizes first (progress printed)."""
import os
import sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05098_b200 import _native, corpus  # noqa: E402

dev = torch.device("cuda", 0)
size = int(sys.argv[1])
profile = sys.argv[2] if len(sys.argv) > 2 else "latin"
d = corpus.generate(profile, size, 2, device=dev)
h_in = torch.empty(size, dtype=torch.uint8).pin_memory()
h_in.copy_(d.cpu())
print("pinned ptr", hex(h_in.data_ptr()), flush=True)
from cuda.bindings import runtime as rt  # noqa: E402
err, attr = rt.cudaPointerGetAttributes(h_in.data_ptr())
print("attrs", err, attr.type, hex(attr.devicePointer), hex(attr.hostPointer), flush=True)
h_out = torch.empty(2 * size, dtype=torch.uint8).pin_memory()
op = _native.OP_UTF8_TO_UTF16LE
ws = torch.empty(_native.workspace_bytes(op, size) // 8 + 1, dtype=torch.int64, device=dev)
res = torch.empty(3, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream(dev)
_native.launch(op, h_in, size, h_out.view(torch.int16), size, ws, res, s)
print("launched", flush=True)
torch.cuda.synchronize()
print("res", res.cpu().tolist(), flush=True)
ref = torch.empty(size, dtype=torch.int16, device=dev)
res2 = torch.empty(3, dtype=torch.int64, device=dev)
_native.launch(op, d, size, ref, size, ws, res2, s)
torch.cuda.synchronize()
w = int(res2[2])
print("same", res.cpu().tolist() == res2.cpu().tolist(), torch.equal(h_out.view(torch.int16)[:w], ref[:w].cpu()), flush=True)
