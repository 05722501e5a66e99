#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma or hub" > gpurun_out/it_t.log 2>&1
tail -3 gpurun_out/it_t.log
rm -f gpurun_out/it_tv.log
for t in 0 2 3; do RPQ_TMA=$t timeout 600 python scripts/time_variant.py rmat24 64 >> gpurun_out/it_tv.log 2>&1; done
RPQ_TMA=2 RPQ_LIB_PATH=build/variants/librpq_t2m5.so timeout 600 python scripts/time_variant.py rmat24 64 >> gpurun_out/it_tv.log 2>&1
for t in 0 2; do RPQ_TMA=$t timeout 600 python scripts/time_variant.py cfg2 >> gpurun_out/it_tv.log 2>&1; done
cut -c1-100 gpurun_out/it_tv.log
