#!/bin/bash
# ncu evidence for profiles/ (run on the B200 through gpurun):
#   launch list of the bench command (cfg2 headline), DRAM traffic per
#   level-kernel launch per workload, and --set full captures of the dense
#   launches of every hot kernel.
# usage: scripts/profile_round.sh TAG
set -x
TAG=$1
O=gpurun_out/prof_$TAG; mkdir -p $O
export RPQ_HOST_LOOP=1   # ncu does not see launches inside the conditional graph body
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-north-star --no-cfg3 > $O/bench_under_ncu_cfg2.log 2>&1
for wl in cfg2 cfg5 cfg3; do
  PROF_NOSTATS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"k_level|k_pull|k_count_total|k_clear_dense" --csv --log-file $O/traffic_$wl.csv \
      python scripts/prof_workload.py $wl > $O/traffic_$wl.log 2>&1
done
F="--set full --clock-control none --import-source on"
PROF_NOSTATS=1 ncu $F -k k_level -s 10 -c 1 -o $O/full_k_level_cfg2 python scripts/prof_cfg2.py "a*" > $O/full1.log 2>&1
PROF_NOSTATS=1 ncu $F -k k_level -s 2 -c 1 -o $O/full_k_level_cfg5 python scripts/prof_workload.py cfg5 > $O/full2.log 2>&1
PROF_NOSTATS=1 ncu $F -k regex:k_level_hub -s 2 -c 1 -o $O/full_k_level_hub_cfg5 python scripts/prof_workload.py cfg5 > $O/full3.log 2>&1
PROF_NOSTATS=1 ncu $F -k regex:k_count_total -c 1 -o $O/full_k_count_total_cfg5 python scripts/prof_workload.py cfg5 > $O/full4.log 2>&1
PROF_PAIRS=1 ncu $F -k regex:k_write_pairs -c 1 -o $O/full_k_write_pairs_cfg2 python scripts/prof_workload.py cfg2 > $O/full5.log 2>&1
PROF_NOSTATS=1 ncu $F -k k_pull -s 1 -c 1 -o $O/full_k_pull_cfg3 python scripts/prof_workload.py cfg3 > $O/full6.log 2>&1
echo done
