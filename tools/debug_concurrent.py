"""Minimal concurrency probe: the TMA stencil on one stream while face
copy kernels run on another stream over unrelated buffers. Any mismatch
against an isolated sweep means kernels interfere."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    mode = sys.argv[4] if len(sys.argv) > 4 else "both"  # both | pack | unpack | none | copy
    g = torch.Generator(device="cuda").manual_seed(3)
    cur = torch.randn((n + 2,) * 3, dtype=torch.float64, device="cuda", generator=g)
    ref = torch.zeros_like(cur)
    s0 = torch.cuda.current_stream().cuda_stream
    box = (1, n + 1, 1, n + 1, k0, n + 1)
    _lib.call("hx_stencil_box", cur.data_ptr(), ref.data_ptr(), n, n, n, *box, None, s0)
    torch.cuda.synchronize()
    other = torch.randn((n + 2,) * 3, dtype=torch.float64, device="cuda", generator=g)
    slot = torch.zeros(n * n * 6, dtype=torch.float64, device="cuda")
    S = torch.cuda.Stream()
    C = torch.cuda.Stream(priority=-1)
    bad_total = 0
    for r in range(reps):
        out = torch.zeros_like(cur)
        torch.cuda.synchronize()
        for _ in range(8):  # keep C busy across the sweep
            for d in range(6):
                if mode in ("both", "pack"):
                    _lib.call("hx_pack", other.data_ptr(), n, n, n, d, slot.data_ptr(), C.cuda_stream)
                if mode in ("both", "unpack"):
                    _lib.call("hx_unpack", other.data_ptr(), n, n, n, d, slot.data_ptr(), C.cuda_stream)
                if mode == "copy":
                    _lib.call("hx_copy_sm", slot.data_ptr(), other.data_ptr(), slot.numel() * 8,
                              C.cuda_stream)
                if mode == "torch":
                    with torch.cuda.stream(C):
                        slot.add_(1.0)
        _lib.call("hx_stencil_box", cur.data_ptr(), out.data_ptr(), n, n, n, *box, None, S.cuda_stream)
        torch.cuda.synchronize()
        bad = int((out != ref).sum().item())
        bad_total += bad
        if bad:
            idx = (out != ref).nonzero()[:4].tolist()
            print(f"rep {r}: {bad} mismatching cells, e.g. {idx}", flush=True)
    print(f"n={n} k0={k0} mode={mode}: total mismatches {bad_total} over {reps} reps", flush=True)


if __name__ == "__main__":
    main()
