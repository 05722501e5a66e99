#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py -q -x -k "hub or tma or rmat24" > gpurun_out/it_t.log 2>&1
tail -2 gpurun_out/it_t.log
rm -f gpurun_out/it_tv.log
for v in hl4096 base hl1024 hl256 hl4096 base; do
  if [ $v = base ]; then L=paper_2602_20748_b200/librpq.so; else L=build/variants/librpq_$v.so; fi
  RPQ_LIB_PATH=$L timeout 600 python scripts/time_variant.py rmat24 64 >> gpurun_out/it_tv.log 2>&1
done
cut -c1-100 gpurun_out/it_tv.log
