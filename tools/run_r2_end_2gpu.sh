# End-of-round 2-GPU set on the final code (gpurun --gpus 2): the multi-GPU and
# cross-process tests, the N = 2 bench lines, small blocks and the z split
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ipc_runtime.py -q > gpurun_out/r2_end_n2_tests.log 2>&1; tail -2 gpurun_out/r2_end_n2_tests.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$R --master-port 29601 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_end_n2.json 2> gpurun_out/r2_end_n2.err
$R --master-port 29602 bench.py --gpus 2 --block 768 --steps 50 --warmup 5 --no-data-alt > gpurun_out/r2_end_n2_768.json 2> gpurun_out/r2_end_n2_768.err
for p in 2 8; do timeout 180 python tools/prof_small.py --pes $p --two-gpus --iters 1000; done > gpurun_out/r2_end_small_2gpu.jsonl 2>&1
timeout 300 python tools/prof_zshell.py --n 1536 --two-gpus > gpurun_out/r2_end_zshell_2gpu.json 2>&1
