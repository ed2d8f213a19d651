"""Can TMA read peer (NVLink) memory? hx_stencil launched on GPU 0 with its
input field on GPU 1 (P2P-mapped): bit-exact vs the same sweep on GPU 1, and
timed (one 768^3 sweep, the whole input crossing NVLink)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2102_12416_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
_lib.call("hx_enable_peer", 0, 1)
_lib.call("hx_enable_peer", 1, 0)
g = torch.Generator(device="cuda:1"); g.manual_seed(0)
cur1 = torch.empty((n + 2,) * 3, dtype=torch.float64, device="cuda:1").normal_(generator=g)
ref1 = torch.zeros_like(cur1)
out0 = torch.zeros((n + 2,) * 3, dtype=torch.float64, device="cuda:0")
_lib.call("hx_set_device", 1)
_lib.call("hx_stencil", cur1.data_ptr(), ref1.data_ptr(), n, n, n, None, torch.cuda.current_stream(1).cuda_stream)
torch.cuda.synchronize(1)
_lib.call("hx_set_device", 0)
s0 = torch.cuda.current_stream(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_lib.call("hx_stencil", cur1.data_ptr(), out0.data_ptr(), n, n, n, None, s0.cuda_stream)
with torch.cuda.device(0):
    e0.record(s0)
    for _ in range(5):
        _lib.call("hx_stencil", cur1.data_ptr(), out0.data_ptr(), n, n, n, None, s0.cuda_stream)
    e1.record(s0)
torch.cuda.synchronize(0)
ms = e0.elapsed_time(e1) / 5
same = torch.equal(out0[1:-1, 1:-1, 1:-1].cpu().view(torch.int64), ref1[1:-1, 1:-1, 1:-1].cpu().view(torch.int64))
print({"n": n, "bitexact_tma_from_peer": same, "ms": ms, "nvlink_read_gbs": 8 * n ** 3 / ms / 1e6,
       "variant": _lib.raw("hx_stencil_last_variant")()})
