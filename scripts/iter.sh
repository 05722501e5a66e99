#!/bin/bash
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/it_tv.log
for wl in cfg2 "rmat24 64"; do
  for v in t2m5 t3m4 t6m2 t8m1; do RPQ_TMA=1 RPQ_LIB_PATH=build/variants/librpq_$v.so timeout 600 python scripts/time_variant.py $wl >> gpurun_out/it_tv.log 2>&1; done
done
cut -c1-100 gpurun_out/it_tv.log
