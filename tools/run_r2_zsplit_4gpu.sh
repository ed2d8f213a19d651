# z splits on 4 GPUs with the interior-sweep z faces (gpurun --gpus 4):
# 3072^3 strong under the reference (1,2,2) and b200 (2,2,1) policies
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$R --master-port 29621 bench.py --gpus 4 --dims 3072,3072,3072 --policy reference --steps 20 --warmup 5 --no-data-alt --no-p2p > gpurun_out/r2_z_n4_strong_reference.json 2> gpurun_out/r2_z_n4_strong_reference.err
$R --master-port 29622 bench.py --gpus 4 --dims 3072,3072,3072 --policy b200 --steps 20 --warmup 5 --no-data-alt --no-p2p > gpurun_out/r2_z_n4_strong_b200.json 2> gpurun_out/r2_z_n4_strong_b200.err
$R --master-port 29623 bench.py --gpus 4 --dims 3072,3072,3072 --policy reference --steps 20 --warmup 5 --no-data-alt --no-p2p > gpurun_out/r2_z_n4_strong_reference2.json 2> gpurun_out/r2_z_n4_strong_reference2.err
timeout 900 python tools/emulate8.py > gpurun_out/r2_z_emulate8.log 2>&1
for f in r2_z_n4_strong_reference r2_z_n4_strong_b200 r2_z_n4_strong_reference2; do
  python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['config']['grid'], d['clocks'])"
done
tail -5 gpurun_out/r2_z_emulate8.log
