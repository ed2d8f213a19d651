# same-box A/B of the persistent small-block kernel on 2 GPUs:
#   bash tools/run_small_ab.sh other_libhx.so   (prof_small 64^3 x 2 / x 8 blocks, 128^3 x 8)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sab_build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "persist or acceptance" > gpurun_out/sab_tests.log 2>&1
echo "tests rc=$?"
for r in 1 2; do
  for lib in paper_2102_12416_b200/libhx.so "$1"; do
    for pes in 2 8; do
      echo "== $lib pes=$pes"
      HX_LIB_PATH=$PWD/$lib timeout 300 python tools/prof_small.py --pes $pes --two-gpus --iters 1000
    done
    echo "== $lib 128 pes=8"
    HX_LIB_PATH=$PWD/$lib timeout 300 python tools/prof_small.py --dims 128,128,128 --pes 8 --two-gpus --iters 500
  done
done
