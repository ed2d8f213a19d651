"""Cross-check Jacobi runs at a large size: sequential GPU sweep vs the halo
engine (1 or 2 GPUs, overlap on/off, both policies) vs the runtime path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2102_12416_b200.halo import HaloJacobi
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    dims = (n, n, n)
    ref, _ = sequential_oracle(dims, iters)
    ngpu = torch.cuda.device_count()
    for gpus in ([0], list(range(min(2, ngpu)))):
        for exchange, overlap in (("p2p", False), ("p2p", True), ("fused", False)):
            for policy in ("reference", "b200"):
                eng = HaloJacobi(dims, 2, device_of=lambda r: gpus[r % len(gpus)], overlap=overlap,
                                 policy=policy, exchange=exchange)
                timing = {}
                for _ in range(iters):
                    eng.step(timing=timing if os.environ.get("TIMING") else None)
                eng.check_errors()
                f = eng.assemble()
                d = np.abs(f - ref)
                bad = np.argwhere(d != 0)
                print(f"gpus={gpus} exchange={exchange} overlap={overlap} policy={policy} grid={eng.grid} "
                      f"max|d|={d.max():.3e} nbad={len(bad)} first={bad[:3].tolist()}", flush=True)
                eng.close()
                del eng
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
