# launch times of the peel kernels over one BERT explore (ncu, serialised)
REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_peel_cmp.csv python scripts/prof_phases.py bert > /dev/null 2>&1
