#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py -q -x -k "sparse or rmat24 or batch or hub or shard or ldbc" > gpurun_out/it_t.log 2>&1
tail -3 gpurun_out/it_t.log
rm -f gpurun_out/it_tv.log
timeout 600 python scripts/time_variant.py rmat24 64 >> gpurun_out/it_tv.log 2>&1
cut -c1-100 gpurun_out/it_tv.log
export RPQ_HOST_LOOP=1 PROF_NOSTATS=1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_level|k_count|k_clear" --csv --log-file gpurun_out/traffic_cfg5_v3.csv python scripts/prof_workload.py cfg5 > gpurun_out/traffic_cfg5_v3.log 2>&1
python scripts/ncu_summary.py traffic gpurun_out/traffic_cfg5_v3.csv
