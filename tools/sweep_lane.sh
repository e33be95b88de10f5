#!/bin/bash
# sweep k_mic_lane2 helper policy (FLIPB200_LANE_MODE) x prefetch depth x tile at 256^3
cd "$(dirname "$0")/.." || exit 1
TILES=${TILES:-"16x16 16x8"}
DEPTHS=${DEPTHS:-"4 8 16"}
MODES=${MODES:-"0 1 2 3"}
for t in $TILES; do for d in $DEPTHS; do for m in $MODES; do
  r=$(FLIPB200_WAVE_TILE=$t FLIPB200_LANE_DEPTH=$d FLIPB200_LANE_MODE=$m timeout 120 python -c "
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name='dam-break', res=256)
st = P.make_scene(spec, 0)
P.step(st, spec); r = P.step(st, spec)
print(round(r.timings.project, 2), r.solver_iterations, r.solver_residual)
" 2>&1 | tail -1)
  echo "tile $t depth $d mode $m: $r"
done; done; done
