cd $GRAFT_REPO_ROOT
for wl in cfg2 "rmat24 64"; do
  for v in base minb4 minb4s16 minb6 minb4h3; do
    RPQ_LIB_PATH=build/variants/librpq_$v.so python scripts/time_variant.py $wl >> gpurun_out/var_r2.txt 2>&1
  done
done
