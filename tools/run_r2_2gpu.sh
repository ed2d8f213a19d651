# 2-GPU measurement set (gpurun --gpus 2): fused-exchange parity, face-kernel A/B, bench N=2
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_scale.py tests/test_gpu_runtime.py -x -q -k "fused or halo or thick" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "fused or engine or graph" 2>&1 | tail -2
for cfg in "1 1" "1 0" "0 1"; do set -- $cfg; HX_SHELL_FACE_TMA=$1 HX_FACE_BULK=$2 python tools/prof_fused.py --n 1536 --reps 10 | sed "s/^/{\"face_tma\": $1, \"bulk\": $2, \"r\": /; s/$/}/"; done > gpurun_out/r2_fused_2gpu.jsonl 2>&1
cut -c1-330 gpurun_out/r2_fused_2gpu.jsonl
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err
tail -2 gpurun_out/r2_bench_n2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench_n2.json").read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ("value","ms_per_step","halo","p2p")})[:3000])
PY
ncu --set full --clock-control none --import-source on -k regex:"face_tma" -c 2 -o gpurun_out/r2_face_2gpu python tools/prof_fused.py --n 1536 --reps 1 --iso-only > /dev/null 2>&1
ls gpurun_out
