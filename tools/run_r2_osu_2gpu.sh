# final OSU sweep on 2 GPUs (API level, persistent channel, device level) + NCCL comparison
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/run_osu.py --out gpurun_out/r2_osu_2gpu.json > gpurun_out/r2_osu_2gpu.log 2>&1
python tools/osu_table.py gpurun_out/r2_osu_2gpu.json > gpurun_out/r2_osu_2gpu_table.md 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/nccl_osu.py --out gpurun_out/r2_nccl_osu_2gpu.json > gpurun_out/r2_nccl_osu_2gpu.log 2>&1
head -30 gpurun_out/r2_osu_2gpu_table.md; tail -5 gpurun_out/r2_nccl_osu_2gpu.log
