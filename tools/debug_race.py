"""Lock-step a sequential single-block sweep and halo engines (overlap on /
off) on one GPU; report the first iteration where an engine diverges."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import HaloJacobi

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    which = sys.argv[3] if len(sys.argv) > 3 else "both"
    engines = {}
    if which in ("both", "overlap"):
        engines["overlap"] = HaloJacobi((n, n, n), 2, device_of=lambda r: 0, overlap=True,
                                       exchange="p2p")
    if which in ("both", "plain"):
        engines["plain"] = HaloJacobi((n, n, n), 2, device_of=lambda r: 0, overlap=False,
                                     exchange="p2p")
    grid = next(iter(engines.values())).grid
    print("grid", grid, flush=True)
    seq = [torch.empty((n + 2,) * 3, dtype=torch.float64, device="cuda") for _ in range(2)]
    s = torch.cuda.current_stream().cuda_stream
    for t in seq:
        _lib.call("hx_init_block", t.data_ptr(), n, n, n, 1, 1.0, 0.0, 0.0, s)
    cur = 0
    for it in range(iters):
        _lib.call("hx_stencil", seq[cur].data_ptr(), seq[cur ^ 1].data_ptr(), n, n, n, None, s)
        cur ^= 1
        torch.cuda.synchronize()
        for name, e in engines.items():
            e.step()
            e.synchronize()
            for comm in e.comm.values():
                comm.synchronize()
            for r, b in e.blocks.items():
                f = b.fields[b.cur][1:-1, 1:-1, 1:-1]
                ix, iy, iz = r % grid[0], (r // grid[0]) % grid[1], r // (grid[0] * grid[1])
                g = seq[cur][1 + ix * b.bx:1 + (ix + 1) * b.bx, 1 + iy * b.by:1 + (iy + 1) * b.by,
                             1 + iz * b.bz:1 + (iz + 1) * b.bz]
                if not torch.equal(f, g):
                    bad = (f != g).nonzero()
                    print(f"{name}: iter {it} rank {r}: {bad.shape[0]} bad; first {bad[:4].tolist()} "
                          f"got {f[tuple(bad[0])].item()} want {g[tuple(bad[0])].item()}", flush=True)
                    del engines[name]
                    break
            else:
                continue
            break
        if not engines:
            return
    print("survivors:", list(engines), flush=True)


if __name__ == "__main__":
    main()
