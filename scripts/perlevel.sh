#!/bin/bash
# Per-launch DRAM bytes and duration of every kernel of one COUNT (and one
# PAIRS) evaluation of the cfg2 queries (development aid; run through gpurun).
cd $GRAFT_REPO_ROOT
O=gpurun_out/perlevel; mkdir -p $O
python scripts/time_variant.py cfg2 > $O/tv_cfg2.txt 2>&1
export RPQ_HOST_LOOP=1 PROF_NOSTATS=1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none --csv --log-file $O/count_cfg2.csv python scripts/prof_workload.py cfg2 > $O/count.log 2>&1
PROF_PAIRS=1 ncu --metrics $M --clock-control none --csv --log-file $O/pairs_cfg2.csv python scripts/prof_workload.py cfg2 > $O/pairs.log 2>&1
echo done
