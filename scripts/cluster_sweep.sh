# wave-loop cluster size / window sweep on BERT: saturate / total ms of the warm repetitions
for cfg in "1 0" "8 1024" "8 2048" "8 4096" "8 8192" "1 0"; do
  set -- $cfg
  echo "nc=$1 win=$2: "; TSAT_WAVE_CLUSTER=$1 TSAT_WAVE_CLUSTER_WIN=$2 REPS=5 python scripts/prof_phases.py bert 2>&1 | grep -E "^\[[2-4]\]|wave-cta" | tail -4
done
