# z-tile L2 promotion A/B (HX_FACE_ZPROMO) on the z split, 1 GPU: bash tools/run_zpromo_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/zp_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_scale.py -x -q > gpurun_out/zp_tests.log 2>&1; echo tests=$?
for r in 1 2; do for zp in 0 3; do echo "== zpromo $zp"; HX_FACE_ZPROMO=$zp timeout 300 python tools/prof_zshell.py --n 1536; done; done
for zp in 0 3; do HX_FACE_ZPROMO=$zp ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:face_tma -c 6 --csv --log-file gpurun_out/zp_ncu_$zp.csv python tools/prof_zshell.py --n 1536 > /dev/null 2>&1; done
