#!/bin/bash
# ncu evidence at the current source tree (run on the GPU box from the repo root):
#   launch lists (time + DRAM bytes + L2 hit per launch) of one BERT bench step and of
#   each configs[4] 10M kernel region, plus --set full captures of the top kernels.
# Usage: scripts/capture_head.sh TAG   -> gpurun_out/TAG/
TAG=${1:-head}
O=gpurun_out/$TAG
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
sha256sum paper_2101_01332_b200/csrc/*.cu paper_2101_01332_b200/csrc/*.cuh > $O/sources.sha256
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches_bert.csv \
    python scripts/prof_bert_window.py > $O/bert.log 2>&1
for r in ematch rebuild_forced rebuild_cascade costs greedy; do
  TSAT_PROF_REGION=$r REPS=1 ncu --profile-from-start off --metrics $M --clock-control none --csv \
      --log-file $O/launches_10m_$r.csv python scripts/synth_sweep.py > $O/10m_$r.log 2>&1
done
if [ -z "$NO_FULL" ]; then
  TSAT_PROF_REGION=ematch REPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none \
      -k regex:k_em_ -o $O/ematch_full python scripts/synth_sweep.py > $O/full_ematch.log 2>&1
  TSAT_PROF_REGION=rebuild_forced REPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none \
      -k regex:k_rebuild -o $O/rebuild_full python scripts/synth_sweep.py > $O/full_rebuild.log 2>&1
  ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_wave_cta -c 3 \
      -o $O/wavecta_full python scripts/prof_bert_window.py > $O/full_wave.log 2>&1
fi
ls -la $O
