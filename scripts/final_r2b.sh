#!/bin/bash
# Round-2 final evidence after the extraction rewrite (one gpurun call): GPU
# test suite, smoke, bench lines (default, per-rank N = 8 share, reference
# arm), compute-sanitizer on the sanitize workload, launch list of the bench
# command, per-kernel DRAM traffic of cfg2 COUNT and PAIRS, and --set full
# captures of the rewritten extraction kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final_r2b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as E; E.smoke(); print('smoke OK')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --sample-shards 8 --no-north-star --no-cfg3 --no-cpu-baseline --no-pairs > $O/bench_cfg2_shard8.json 2> $O/bench_shard8.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py > $O/sanitize_$t.log 2>&1
  tail -1 $O/sanitize_$t.log
done
export RPQ_HOST_LOOP=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-north-star --no-cfg3 > $O/bench_under_ncu.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
PROF_NOSTATS=1 ncu --metrics $M --clock-control none --csv --log-file $O/traffic_count_cfg2.csv python scripts/prof_workload.py cfg2 > $O/traffic_count.log 2>&1
PROF_PAIRS=1 ncu --metrics $M --clock-control none --csv --log-file $O/traffic_pairs_cfg2.csv python scripts/prof_workload.py cfg2 > $O/traffic_pairs.log 2>&1
F="--set full --clock-control none --import-source on"
PROF_PAIRS=1 ncu $F -k regex:k_write_pairs -c 1 -o $O/full_k_write_pairs_cfg2 python scripts/prof_workload.py cfg2 > $O/full_wp.log 2>&1
PROF_PAIRS=1 ncu $F -k regex:k_tile_counts -c 1 -o $O/full_k_tile_counts_cfg2 python scripts/prof_workload.py cfg2 > $O/full_tc.log 2>&1
ls $O
