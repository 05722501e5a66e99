#!/bin/bash
# ncu evidence for profiles/ (run on the B200 through gpurun):
#   launch list of the bench command (cfg2), DRAM traffic per k_level launch
#   and one --set full capture of a dense k_level launch, per workload.
# usage: scripts/profile_round.sh TAG "cfg2 cfg5 cfg3"
set -x
TAG=$1; WLS=${2:-"cfg2 cfg5 cfg3"}
O=gpurun_out/prof_$TAG; mkdir -p $O
export RPQ_HOST_LOOP=1   # ncu does not see launches inside the conditional graph body
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu_cfg2.log 2>&1
for wl in $WLS; do
  PROF_NOSTATS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k_level --csv --log-file $O/traffic_$wl.csv \
      python scripts/prof_workload.py $wl > $O/traffic_$wl.log 2>&1
done
# dense mid-traversal levels: cfg2 a* level 10, cfg5 first batch level 3, cfg3 knows+ level 2
PROF_NOSTATS=1 ncu --set full --clock-control none --import-source on -k k_level -s 10 -c 1 -o $O/full_cfg2 \
    python scripts/prof_cfg2.py "a*" > $O/full_cfg2.log 2>&1
PROF_NOSTATS=1 ncu --set full --clock-control none --import-source on -k k_level -s 2 -c 1 -o $O/full_cfg5 \
    python scripts/prof_workload.py cfg5 > $O/full_cfg5.log 2>&1
echo done
