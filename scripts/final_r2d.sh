#!/bin/bash
# Round-2 closing evidence (one gpurun call): GPU test suite, smoke, bench
# lines (default, per-rank N = 8 share, reference arm) with the group-aligned
# batch planner.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final_r2d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as E; E.smoke(); print('smoke OK')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --sample-shards 8 --no-north-star --no-cfg3 --no-cpu-baseline --no-pairs > $O/bench_cfg2_shard8.json 2> $O/bench_shard8.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
ls $O
