# face-kernel store variants on 2 GPUs (HX_FACE_BULK: 0 plain, 1 bulk copy, 2 paired 16-B stores)
python -c "import __graft_entry__ as g; g.build()"
for b in 0 1 2; do HX_FACE_BULK=$b timeout 120 python tools/dbg_face.py 2>&1 | tail -1; done
for cfg in "1 2" "1 1" "1 0" "0 0"; do set -- $cfg; HX_SHELL_FACE_TMA=$1 HX_FACE_BULK=$2 python tools/prof_fused.py --n 1536 --reps 10 --iso-only | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['shell_alone']['ms'], d['shell_alone']['nvlink_gbs'])"; done
for m in 2 4; do HX_FACE_GRID_MULT=$m HX_FACE_BULK=2 python tools/prof_fused.py --n 1536 --reps 10 --iso-only | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mult $m', d['shell_alone']['ms'], d['shell_alone']['nvlink_gbs'])"; done
