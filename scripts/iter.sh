#!/bin/bash
# development iteration (one gpurun call): parity of what changed + timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_dist.py "tests/test_gpu_exact.py::test_cfg2_pairs_of_2048_sources" -q -x > gpurun_out/it_t.log 2>&1
tail -3 gpurun_out/it_t.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-north-star --no-cfg3 --no-cpu-baseline > gpurun_out/it_b.json 2> gpurun_out/it_b.err
python -c "import json; d=json.loads(open('gpurun_out/it_b.json').read().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['pairs_mode'])"
rm -f gpurun_out/it_tv.log
for wl in cfg2 "rmat24 64"; do
  timeout 600 python scripts/time_variant.py $wl >> gpurun_out/it_tv.log 2>&1
  RPQ_LIB_PATH=build/variants/librpq_minb4.so timeout 600 python scripts/time_variant.py $wl >> gpurun_out/it_tv.log 2>&1
done
cut -c1-100 gpurun_out/it_tv.log
