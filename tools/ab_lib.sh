# same-box A/B of two libhx builds on the power-probe workload: bash tools/ab_lib.sh other.so
python -c "import __graft_entry__ as g; g.build()"
for r in 1 2; do
  for lib in paper_2102_12416_b200/libhx.so "$1"; do
    echo "== $lib"; HX_LIB_PATH=$PWD/$lib python tools/data_dependence.py 1536 power 2>&1 | head -2
  done
done
