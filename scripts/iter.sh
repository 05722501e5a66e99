#!/bin/bash
cd $GRAFT_REPO_ROOT
export RPQ_HOST_LOOP=1 PROF_NOSTATS=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_level$" -s 2 -c 1 -o gpurun_out/full_sh8_l2 python scripts/prof_workload.py cfg2 8 > gpurun_out/f1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_level$" -s 8 -c 1 -o gpurun_out/full_sh8_l8 python scripts/prof_workload.py cfg2 8 > gpurun_out/f2.log 2>&1
