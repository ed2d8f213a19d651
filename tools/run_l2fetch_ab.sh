# L2 fetch granularity A/B (HX_L2_FETCH, cudaLimitMaxL2FetchGranularity) on the
# z-face paths and the stencil: bash tools/run_l2fetch_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2f_build.log 2>&1
for f in "" 32 64 128; do
  echo "== HX_L2_FETCH=$f"
  env ${f:+HX_L2_FETCH=$f} timeout 300 python tools/prof_faces.py --n 1536 | grep '"dir": [45]'
  env ${f:+HX_L2_FETCH=$f} timeout 300 python tools/prof_zshell.py --n 1536
done
for f in 32 128; do
  HX_L2_FETCH=$f ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:face_tma -c 4 --csv --log-file gpurun_out/l2f_ncu_$f.csv python tools/prof_zshell.py --n 1536 > /dev/null 2>&1
done
