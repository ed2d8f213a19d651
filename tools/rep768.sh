#!/bin/bash
# Repeat the 768^3-per-GPU N=4 bench (variance check); optional env passes through.
for r in 1 2 3; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29800 + r)) bench.py --gpus 4 --block 768 --no-e2e --no-cpu-baseline 2>/dev/null \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']; print('$TAG', round(d['value'],1), round(d['ms_per_step'],4), round(h['exchange_ms'],4), round(h['exposed_ms'],4), round(h['interior_ms'],4))"
done
