import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2102_12416_b200.halo import HaloJacobi
from oracle import jacobi_np
dims=(64,32,400)
for bulk in ("0","1"):
    os.environ["HX_FACE_BULK"]=bulk
    eng = HaloJacobi(dims, 2, device_of=lambda r: 0, exchange="fused")
    eng.run(5); eng.check_errors()
    want,_ = jacobi_np.sequential(dims, 5)
    print("bulk", bulk, eng.assemble().tobytes()==want.tobytes(), flush=True)
