#!/bin/bash
# parity-split leaf-up GEMM: parity (c0 suite incl. many RHS, q = 14 live oracle, c3 full-mesh poles), c3 / c1 bench
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "config0 or ragged" 2>&1 | tail -4 > $O/eo_tests.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "64rhs or n4_p16 or c1" 2>&1 | grep -E "rel L2|passed|failed" | cut -c1-200 >> $O/eo_tests.txt
cat $O/eo_tests.txt
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/eo_bench_c3.log 2>&1
timeout 600 python bench.py --config c1_rsw_16x16_p16 --steps 50 --no-cpu-baseline > $O/eo_bench_c1.log 2>&1
for f in $O/eo_bench_c3.log $O/eo_bench_c1.log; do echo $f; tail -1 $f | python -c "
import sys, json
try:
    d = json.loads(sys.stdin.read())
    print(d['value'], d['ms_per_step'])
    print({k: v['ms_per_step'] for k, v in d['roofline']['per_class'].items()}, d['roofline']['whole_step'])
except Exception as e:
    print('ERR', e)
"; done
