#!/bin/bash
# batched spectral pre/back kernels: parity (c0 suite + q=14 live-oracle case), then c3 / c1 bench lines
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "config0 or ragged or sharded" 2>&1 | tail -4 > $O/b_tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "n4_p16" 2>&1 | tail -3 >> $O/b_tests.txt
cat $O/b_tests.txt
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/b_bench_c3.log 2>&1
timeout 600 env REXP_LANES=2 python bench.py --steps 20 --no-cpu-baseline > $O/b_bench_c3_lanes2.log 2>&1
timeout 600 python bench.py --config c1_rsw_16x16_p16 --steps 50 --no-cpu-baseline > $O/b_bench_c1.log 2>&1
for f in $O/b_bench_*.log; do echo $f; tail -1 $f | python -c "
import sys, json
try:
    d = json.loads(sys.stdin.read())
    print(d['value'], d['ms_per_step'])
    print({k: v['ms_per_step'] for k, v in d['roofline']['per_class'].items()})
except Exception as e:
    print('ERR', e)
"; done
