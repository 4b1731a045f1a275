# hashcons load-factor sweep: configs[4] kernels (ms) and BERT step
for l in 0.5 0.75; do
  echo "== load $l"
  TSAT_HC_LOAD=$l REPS=2 python scripts/synth_sweep.py 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print({k: round(d[k]['ms'],3) for k in ['ematch_13','rebuild_forced','rebuild_cascade','costs','greedy','apply_wave']}, 'search', [round(x*1e3,1) for x in d['search_s']])"
  TSAT_HC_LOAD=$l REPS=3 python scripts/prof_phases.py bert 2>&1 | grep "^\[2\]"
done
