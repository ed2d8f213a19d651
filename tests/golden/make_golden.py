"""Generate golden vectors by importing the reference itself.

Run IN THE DEV CONTAINER only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports charmlet read-only from /root/reference/pkg/src and freezes:
  * sequential_oracle((64,64,64),100): sha256, sum, full residual history
    (cl/jacobi3d.py:181-200) and the full 16^3 x 8 field;
  * run_jacobi fields (sha256) for every mode at small sizes and 1/2/4/8 PEs
    (cl/jacobi3d.py:335-379);
  * _BlockCore.pack outputs and unpack_all results on seeded random fields
    (cl/jacobi3d.py:157-163);
  * one _BlockCore.update step on a seeded random field (cl/jacobi3d.py:165-173);
  * decompose / neighbor_table tables (cl/jacobi3d.py:62-97);
  * tag codec examples (cl/tags.py:81-125) and the OSU payload pattern
    (cl/bench.py:36-37).
Outputs: tests/golden/golden.json and tests/golden/golden.npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from charmlet import jacobi3d as J  # noqa: E402
from charmlet.bench import _pattern  # noqa: E402
from charmlet.config import RuntimeConfig  # noqa: E402
from charmlet.tags import DEVICE, TagLayout  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class _Buf:
    """Host stand-in for a device buffer: _BlockCore only calls .view()."""

    def __init__(self, n):
        self.b = bytearray(n)

    def view(self, dtype, shape):
        return np.frombuffer(self.b, dtype=dtype).reshape(shape)


def main():
    out: dict = {}
    arrays: dict = {}

    # 1. sequential oracle, config C1
    f, res = J.sequential_oracle((64, 64, 64), 100)
    out["seq_64_100"] = {
        "sha256": sha(f), "sum": float(f.sum()),
        "residuals_hex": [float(r).hex() for r in res],
    }
    f16, res16 = J.sequential_oracle((16, 16, 16), 8)
    arrays["seq_16_8"] = f16
    out["seq_16_8_residuals_hex"] = [float(r).hex() for r in res16]
    f_odd, _ = J.sequential_oracle((12, 10, 14), 7, hot=0.75, background=0.125, fill=0.5)
    arrays["seq_12x10x14_7_custom"] = f_odd

    # 2. run_jacobi across modes and PE counts (fields must equal the oracle)
    runs = {}
    for dims, iters, pes_list in (((16, 16, 16), 5, (1, 2, 4, 8)),
                                  ((32, 32, 32), 20, (2, 4))):
        for pes in pes_list:
            for mode in J.MODES:
                r = J.run_jacobi(dims=dims, iters=iters, mode=mode, pes=pes)
                runs[f"{dims[0]}x{dims[1]}x{dims[2]}/{iters}/{pes}/{mode}"] = sha(r["field"])
    out["run_jacobi_sha256"] = runs
    out["seq_sha256"] = {"16x16x16/5": sha(J.sequential_oracle((16,) * 3, 5)[0]),
                         "32x32x32/20": sha(J.sequential_oracle((32,) * 3, 20)[0])}

    # 3. pack / unpack / update on seeded random fields
    for tag, dims, grid, rank in (("a", (12, 10, 16), (2, 2, 2), 0),
                                  ("b", (18, 14, 22), (3, 1, 2), 4),
                                  ("c", (8, 8, 8), (2, 2, 2), 7)):
        core = J._BlockCore(dims, grid, rank, lambda n: _Buf(n))
        rng = np.random.default_rng(sum(map(ord, tag)))
        cur = core._views[core.cur]
        cur[:] = rng.standard_normal(cur.shape)
        arrays[f"pack_{tag}_field"] = cur.copy()
        for d in core.nbr_dirs:
            core.pack(d)
            arrays[f"pack_{tag}_face{d}"] = core._sview[d].copy()
        for p in (0, 1):
            for d in core.nbr_dirs:
                core._rview[p][d][:] = rng.standard_normal(core.face_shape[d])
        core.unpack_all(1)
        arrays[f"unpack_{tag}_field"] = cur.copy()
        for d in core.nbr_dirs:
            arrays[f"unpack_{tag}_rstage{d}"] = core._rview[1][d].copy()
        core.update()
        arrays[f"update_{tag}_next"] = core._views[core.cur].copy()
        out[f"block_{tag}"] = {"dims": dims, "grid": grid, "rank": rank,
                               "nbr_dirs": core.nbr_dirs, "neighbors": core.neighbors,
                               "face_shape": core.face_shape, "face_bytes": core.face_bytes}

    # 4. decomposition and topology
    dec = {}
    for dims in ((64, 64, 64), (128, 64, 64), (96, 48, 24), (7, 7, 7)):
        for n in range(1, 65):
            try:
                dec[f"{dims}/{n}"] = list(J.decompose(dims, n))
            except J.JacobiError:
                dec[f"{dims}/{n}"] = None
    for dims, n in (((3072, 1536, 1536), 2), ((3072, 3072, 1536), 4), ((3072,) * 3, 8),
                    ((3072,) * 3, 4), ((1536, 768, 768), 2), ((1536, 1536, 768), 4),
                    ((1536,) * 3, 8), ((1536,) * 3, 1), ((768,) * 3, 1)):
        dec[f"{dims}/{n}"] = list(J.decompose(dims, n))
    out["decompose"] = dec
    out["neighbors"] = {f"{g}": [J.neighbor_table(g, r) for r in range(g[0] * g[1] * g[2])]
                        for g in ((2, 2, 2), (3, 3, 3), (1, 2, 2), (2, 1, 1), (4, 1, 2))}

    # 5. tags and OSU payload
    lay = TagLayout()
    out["tags"] = {
        "channel": [[cid, d, c, lay.encode_channel(cid, d, c)]
                    for cid, d, c in ((0, 0, 0), (1, 0, 2), (1, 1, 2), (4097, 1, 77))],
        "messaging": [[DEVICE, pe, c, lay.encode_messaging(DEVICE, pe, c)]
                      for pe, c in ((3, 5), (0, 0), (7, 123456))],
        "digest": lay.digest(),
    }
    out["pattern_sha256"] = {str(s): hashlib.sha256(_pattern(s)).hexdigest()
                             for s in (1, 8, 1000, 4096, 65536, 1 << 20)}
    out["generated_from"] = "/root/reference/pkg/src/charmlet (imported read-only)"
    out["reference_cfg_time_mode_default"] = RuntimeConfig().time_mode

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", len(arrays), "arrays;", len(runs), "run_jacobi hashes")


if __name__ == "__main__":
    main()
