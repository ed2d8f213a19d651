#!/bin/bash
# Round-end measurement set: bench lines for every config BASELINE.json names
# that fits the box, the reference arm, and the N=1 ncu launch list.
# usage: tools/run_final.sh TAG NGPU   (writes gpurun_out/TAG_*.json)
tag=$1; ngpu=${2:-4}
mkdir -p gpurun_out
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 \
         --master-port $((29700 + RANDOM % 200)) bench.py --gpus "$@"; }
python bench.py 2> gpurun_out/${tag}_n1.err | grep '^{' > gpurun_out/${tag}_n1.json
python bench.py --impl reference 2> gpurun_out/${tag}_ref.err | grep '^{' > gpurun_out/${tag}_ref.json
if [ "$ngpu" -ge 2 ]; then
  tr 2 2> gpurun_out/${tag}_n2.err | grep '^{' > gpurun_out/${tag}_n2.json
fi
if [ "$ngpu" -ge 4 ]; then
  tr 4 2> gpurun_out/${tag}_n4.err | grep '^{' > gpurun_out/${tag}_n4.json
  tr 4 --block 768 2> gpurun_out/${tag}_n4_768.err | grep '^{' > gpurun_out/${tag}_n4_768.json
  tr 4 --dims 3072,3072,3072 2> gpurun_out/${tag}_n4_strong.err | grep '^{' > gpurun_out/${tag}_n4_strong.json
fi
python bench.py --block 768 --no-cpu-baseline 2> gpurun_out/${tag}_n1_768.err | grep '^{' > gpurun_out/${tag}_n1_768.json
if [ "$ngpu" -ge 2 ]; then
  CUDA_VISIBLE_DEVICES=0,1 python tools/run_osu.py --out gpurun_out/${tag}_osu.json > gpurun_out/${tag}_osu.log 2>&1
fi
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-p2p \
  --no-cpu-baseline > gpurun_out/${tag}_ncu_launches.log 2>&1
for f in gpurun_out/${tag}_*.json; do
  python -c "
import json,sys
try:
    d=json.load(open('$f'))
except Exception as e:
    print('$f', 'EMPTY/FAILED'); sys.exit()
e=d.get('e2e') or {}
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), e.get('value'))
"
done
