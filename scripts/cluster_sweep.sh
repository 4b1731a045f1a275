# wave-loop cluster size sweep on BERT: saturate / total ms of the warm repetition
for nc in 1 8; do echo -n "nc=$nc: "; TSAT_WAVE_CLUSTER=$nc REPS=3 python scripts/prof_phases.py bert 2>&1 | grep "^\[2\]" ; done
