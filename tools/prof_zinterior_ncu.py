"""Four fused steps of a z split (two 1536^3 blocks on one GPU), for ncu:
    ZINT=1|0 ncu ... python tools/prof_zinterior_ncu.py  (z faces from the interior sweep, or slots)"""
import sys, os
sys.path.insert(0, "/root/repo")
from paper_2102_12416_b200.halo import HaloJacobi
n = 1536
eng = HaloJacobi((n, n, 2 * n), 2, device_of=lambda r: 0, exchange="fused", policy="reference")
eng.z_from_interior = os.environ.get("ZINT", "1") == "1"
for _ in range(4):
    eng.step()
eng.synchronize(); eng.check_errors(); eng.close()
