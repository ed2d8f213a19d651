# every face inside the interior sweep (--sweep-exchange 1) vs the boundary
# kernel for x / y faces (0), same box: bash tools/run_sweepx_ab.sh NGPU [BLOCK]
n=${1:-2}
blk=${2:-1536}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
p=29700
for r in 1 2; do
  for sx in 0 1; do
    p=$((p+1))
    $R --master-port $p bench.py --gpus $n --block $blk --steps 50 --warmup 5 --no-data-alt --no-p2p --sweep-exchange $sx > gpurun_out/sx_${n}_${blk}_${sx}_$r.json 2> gpurun_out/sx_${n}_${blk}_${sx}_$r.err
    python -c "import json; d=json.loads(open('gpurun_out/sx_${n}_${blk}_${sx}_$r.json').read().strip().splitlines()[-1]); print('sweep_exchange=$sx', d['value'], d['ms_per_step'], d['halo']['interior_ms'], d['halo']['exposed_ms'], d['gpu_launches'])"
  done
done
