"""Interior-box sweeps as the fused exchange launches them: the whole block
vs boxes trimmed by a -z neighbour (first column k = 2) or a +z neighbour,
on a 1536^3 block, CUDA-event timed (best of 7).

    python tools/prof_box.py [--n 1536]    (HX_TMA_KEEP_GRID=0: the old 68-wide shifted box)
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2102_12416_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    n = ap.parse_args().n
    cur = torch.zeros((n + 2,) * 3, dtype=torch.float64, device="cuda")
    nxt = torch.zeros_like(cur)
    s = torch.cuda.current_stream().cuda_stream
    out = {"n": n, "keep_grid": os.environ.get("HX_TMA_KEEP_GRID", "1")}
    boxes = {"full": (1, n + 1, 1, n + 1, 1, n + 1), "minus_z": (1, n + 1, 1, n + 1, 2, n + 1),
             "plus_z": (1, n + 1, 1, n + 1, 1, n), "both_z": (1, n + 1, 1, n + 1, 2, n),
             "minus_y_minus_z": (1, n + 1, 2, n + 1, 2, n + 1)}
    for name, b in boxes.items():
        ts = []
        for _ in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("hx_stencil_box", cur.data_ptr(), nxt.data_ptr(), n, n, n, *b, None, s)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        cells = (b[1] - b[0]) * (b[3] - b[2]) * (b[5] - b[4])
        ms = min(ts[1:])
        out[name] = {"ms": ms, "gbs": 16 * cells / ms / 1e6}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
