# z faces from the interior sweep: single launch (default) vs split strips
# (HX_ZE_STRIPS=1) vs slots, on one and two GPUs: bash tools/run_zint_ab.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_runtime.py -x -q -k "z_faces or fused or soak" 2>&1 | tail -1
for r in 1 2; do
  for st in 0 1; do
    echo "== HX_ZE_STRIPS=$st"
    HX_ZE_STRIPS=$st timeout 300 python tools/prof_zshell.py --n 1536
    HX_ZE_STRIPS=$st timeout 300 python tools/prof_zshell.py --n 1536 --two-gpus
  done
done
