#!/bin/bash
# Compare halo exchange implementations under torchrun: bench.py lines for
# each (block edge, exchange) pair, one JSON line per run in gpurun_out/.
# usage: tools/cmp_exchange.sh NGPU "1536 768" "p2p fused"
n=$1; blocks=$2; modes=$3
mkdir -p gpurun_out
port=29600
for blk in $blocks; do
  for ex in $modes; do
    port=$((port + 1))
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus "$n" --block "$blk" --exchange "$ex" --no-e2e \
      --no-cpu-baseline 2> "gpurun_out/cmp_${n}_${blk}_${ex}.err" | grep '^{' > "gpurun_out/cmp_${n}_${blk}_${ex}.json"
    python - "$n" "$blk" "$ex" <<'PY'
import json, sys
n, blk, ex = sys.argv[1:]
try:
    d = json.load(open(f"gpurun_out/cmp_{n}_{blk}_{ex}.json"))
except Exception as e:
    print(n, blk, ex, "FAILED", e); sys.exit()
h = d["halo"] or {}
print(f"N={n} block={blk} {ex:6s} {d['value']:8.1f} GLUP/s  {d['ms_per_step']:.4f} ms/step  "
      f"interior {h.get('interior_ms', 0):.4f}  exch {h.get('exchange_ms', 0):.4f}  "
      f"exposed {h.get('exposed_ms', 0):.4f}  frac {d['roofline']['frac']:.4f}")
PY
  done
done
