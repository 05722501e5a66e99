#!/bin/bash
# One GPU call: full gpu test suite, smoke, bench (headline + north star + cfg3),
# a per-rank N=8 share of the headline, and the dense-level ncu captures.
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q --durations=30 > gpurun_out/t4.log 2>&1
python -c "import __graft_entry__ as E; E.smoke()" > gpurun_out/smoke4.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/b4.json 2> gpurun_out/b4.err
python bench.py --steps 10 --warmup 3 --sample-shards 8 --no-north-star --no-cfg3 --no-cpu-baseline --no-pairs > gpurun_out/b4_s8.json 2> gpurun_out/b4_s8.err
O=gpurun_out/prof_r2; mkdir -p $O
export RPQ_HOST_LOOP=1
F="--set full --clock-control none --import-source on"
PROF_NOSTATS=1 ncu $F -k k_level -s 10 -c 1 -o $O/full_k_level_cfg2 python scripts/prof_cfg2.py "a*" > $O/full1.log 2>&1
PROF_NOSTATS=1 ncu $F -k k_level -s 2 -c 1 -o $O/full_k_level_cfg5 python scripts/prof_workload.py cfg5 > $O/full2.log 2>&1
PROF_NOSTATS=1 ncu $F -k k_pull -s 1 -c 1 -o $O/full_k_pull_cfg3 python scripts/prof_workload.py cfg3 > $O/full6.log 2>&1
PROF_PAIRS=1 ncu $F -k k_write_pairs -c 1 -o $O/full_k_write_pairs_cfg2_v2 python scripts/prof_workload.py cfg2 > $O/full5b.log 2>&1
PROF_NOSTATS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_level|k_count|k_clear" --csv --log-file $O/traffic_cfg5_v2.csv python scripts/prof_workload.py cfg5 > $O/traffic_cfg5_v2.log 2>&1
tail -3 gpurun_out/t4.log
