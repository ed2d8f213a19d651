#!/bin/bash
# Fused-shell grid size (CTAs per SM) at N GPUs, 1536^3 per GPU (bench.py, fused exchange).
# usage: tools/sweep_shell_grid.sh N "1 2 4"
n=$1; mults=${2:-"1 2 4"}
for m in $mults; do
  HX_SHELL_GRID_MULT=$m python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" \
    --master-addr 127.0.0.1 --master-port $((29900 + m)) bench.py --gpus "$n" --no-e2e \
    --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']; print('mult=$m', round(d['value'],1), round(d['ms_per_step'],4), round(h['exchange_ms'],4), round(h['interior_ms'],4), 'isolated', round(h['isolated_exchange_ms'],4), round(h['isolated_nvlink_frac'],3))"
done
