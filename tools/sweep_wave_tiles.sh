#!/bin/bash
# quick sweep of wavefront tile shapes / publish periods at 256^3 (2 steps each)
cd "$(dirname "$0")/.." || exit 1
for t in 16x8 16x16 8x8; do
  for p in 2; do
    r=$(FLIPB200_WAVE_TILE=$t FLIPB200_WAVE_PUB=$p timeout 120 python -c "
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name='dam-break', res=256)
st = P.make_scene(spec, 0)
P.step(st, spec); r = P.step(st, spec)
print(round(r.timings.project, 2), r.solver_iterations, r.solver_residual)
" 2>&1 | tail -1)
    echo "tile $t pub $p: $r"
  done
done
