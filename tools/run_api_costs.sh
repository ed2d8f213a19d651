# API-level cost split (1 or 2 GPUs): per-message host time and C-call time
python -c "import __graft_entry__ as g; g.build()"
for api in charm-channel charm-messaging mpi; do
  python tools/prof_api_lat.py --api $api --size 8 --iters 2000
  python tools/prof_api_lat.py --api $api --size 4194304 --iters 3 --bw
done
python tools/prof_api_cprofile.py charm-channel 8 2000 | head -40
