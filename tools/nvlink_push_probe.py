"""NVLink one-way bandwidth for one halo-face-sized message (18.9 MB) on 2
GPUs: copy engine vs SM push vs SM pull, window 1 and 8 (CUDA-graph timed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200 import osu

size = 1536 * 1536 * 8
for window in (1, 8):
    for engine in ("ce", "sm-window", "sm-pull-window"):
        r = osu.device_bandwidth(size, window=window, iters=10, engine=engine)
        print(json.dumps({"size": size, "window": window, "engine": engine,
                          "gbs": r["value_gbps"], "verified": r["verified"]}), flush=True)
