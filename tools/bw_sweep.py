"""Device-level NVLink bandwidth sweep (grid size x engine) at 4 MiB."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import device_bandwidth  # noqa: E402

for size in (1 << 20, 4 << 20, 16 << 20):
    for engine in ("sm-window", "sm-pull-window"):
        r = device_bandwidth(size, window=64, iters=5, engine=engine)
        r["grid_mult"] = os.environ.get("HX_COPY_GRID_MULT", "2")
        print(json.dumps(r), flush=True)
