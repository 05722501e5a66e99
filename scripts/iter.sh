#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "edgeless or many_state or redo or degenerate" > gpurun_out/it_t.log 2>&1
tail -2 gpurun_out/it_t.log
timeout 1200 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r2c.json').read().splitlines()[-1])
ns=d['north_star']; print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], ns['ms'], ns['pe_per_s'], ns['count_ok'], ns['roofline']['frac'], ns['roofline']['ncu_dram_over_algorithmic'])"
