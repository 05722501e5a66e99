#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_dist.py tests/test_gpu_targets.py tests/test_gpu_crpq.py "tests/test_gpu_exact.py::test_cfg2_pairs_of_2048_sources" -q -x > gpurun_out/it_t.log 2>&1
tail -3 gpurun_out/it_t.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-north-star --no-cfg3 --no-cpu-baseline > gpurun_out/it_b.json 2> gpurun_out/it_b.err
python -c "import json; d=json.loads(open('gpurun_out/it_b.json').read().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['pairs_mode'])"
O=gpurun_out/pairsprof; mkdir -p $O
export RPQ_HOST_LOOP=1
PROF_PAIRS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_write_pairs|k_tile_counts" --csv --log-file $O/launches_pairs_v4.csv python scripts/prof_workload.py cfg2 > $O/l.log 2>&1
grep -h k_write_pairs $O/launches_pairs_v4.csv | head -12 | cut -c1-60,200-
