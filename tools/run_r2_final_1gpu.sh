# Round-2 1-GPU end-of-round set: smoke, pytest -m gpu, bench N=1 (driver command), reference arm, ncu launch list
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_end_n1.json 2> gpurun_out/r2_end_n1.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_end_ref.json 2> gpurun_out/r2_end_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e-api > gpurun_out/r2_ncu_bench.log 2>&1
python - <<'PY'
import json
for f in ("r2_end_n1", "r2_end_ref"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, json.dumps({k: d.get(k) for k in ("value", "ms_per_step", "roofline", "clocks", "e2e", "data_alt", "e2e_api", "cpu_baseline", "gpu_launches")})[:3000])
PY
