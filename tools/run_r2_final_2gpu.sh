# Round-2 2-GPU measurement set (gpurun --gpus 2)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ipc_runtime.py -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_n2.json 2> gpurun_out/r2_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 2 --block 768 --steps 50 --warmup 5 --no-data-alt > gpurun_out/r2_n2_768.json 2> gpurun_out/r2_n2_768.err
for p in 2 8; do timeout 180 python tools/prof_small.py --pes $p --two-gpus; done > gpurun_out/r2_small_2gpu.jsonl 2>&1
timeout 300 python tools/prof_zshell.py --n 1536 --two-gpus > gpurun_out/r2_zshell_2gpu.json 2>&1
for api in charm-channel charm-messaging mpi; do
  timeout 300 python tools/prof_api_lat.py --api $api --size 8 --iters 2000
  timeout 300 python tools/prof_api_lat.py --api $api --size 4194304 --iters 3 --bw
done > gpurun_out/r2_api_costs_2gpu.txt 2>&1
timeout 900 python tools/run_osu.py --out gpurun_out/r2_osu_2gpu.json > gpurun_out/r2_osu_2gpu.log 2>&1; python tools/osu_table.py gpurun_out/r2_osu_2gpu.json > gpurun_out/r2_osu_2gpu_table.md 2>&1
ls gpurun_out
