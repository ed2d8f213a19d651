#!/bin/bash
# L2-promotion / grouping / chunk sweep of the TMA stencil (tools/prof_stencil.py).
# usage: tools/sweep_tma_knobs.sh [shape...]   (default 1536^3)
shapes=${@:-1536,1536,1536}
for shape in $shapes; do
  for promo in 1 2 3; do for rep in 1 2; do
    r=$(HX_TMA_L2PROMO=$promo python tools/prof_stencil.py --shape $shape --reps 8 | tail -1)
    echo "shape=$shape promo=$promo rep=$rep $r"
  done; done
done
