#!/bin/bash
# Round-2 evidence in one gpurun call: GPU test suite, smoke, bench lines
# (default = cfg2 headline + RMAT-24 north star + cfg3 + PAIRS + CPU baseline;
# the per-rank N = 8 share; the reference arm), compute-sanitizer on the
# sanitize workload, and the ncu captures of scripts/profile_round.sh.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final_r2; mkdir -p $O
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
bash scripts/profile_round.sh r2 > $O/profile_round.log 2>&1
ls gpurun_out/prof_r2
