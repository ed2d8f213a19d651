# Round-2 4-GPU measurement set (gpurun --gpus 4)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ipc_runtime.py -x -q > gpurun_out/r2_n4_tests.log 2>&1; echo "multi-GPU tests rc=$?"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$R --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_n4.json 2> gpurun_out/r2_n4.err
$R --master-port 29612 bench.py --gpus 4 --block 768 --steps 50 --warmup 5 --no-data-alt > gpurun_out/r2_n4_768.json 2> gpurun_out/r2_n4_768.err
$R --master-port 29613 bench.py --gpus 4 --dims 3072,3072,3072 --policy b200 --steps 20 --warmup 5 --no-data-alt --no-p2p > gpurun_out/r2_n4_strong_b200.json 2> gpurun_out/r2_n4_strong_b200.err
$R --master-port 29614 bench.py --gpus 4 --dims 3072,3072,3072 --policy reference --steps 20 --warmup 5 --no-data-alt --no-p2p > gpurun_out/r2_n4_strong_reference.json 2> gpurun_out/r2_n4_strong_reference.err
python - <<'PY'
import json
for f in ("r2_n4", "r2_n4_768", "r2_n4_strong_b200", "r2_n4_strong_reference"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, json.dumps({k: d.get(k) for k in ("value", "ms_per_step", "config", "halo", "p2p")})[:1500])
    except Exception as e:
        print(f, "ERR", e)
PY
ls gpurun_out
