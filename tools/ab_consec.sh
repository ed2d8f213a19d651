# same-box A/B: consecutive-row stencil (libhx.so) vs the strided-row build (libhx_rowsplit.so)
python -c "import __graft_entry__ as g; g.build()"
for r in 1 2; do
  for lib in paper_2102_12416_b200/libhx.so paper_2102_12416_b200/libhx_rowsplit.so; do
    echo "== $lib"; HX_LIB_PATH=$PWD/$lib python tools/data_dependence.py 1536 power 2>&1 | head -2
  done
done
