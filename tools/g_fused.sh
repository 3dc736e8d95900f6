#!/bin/bash
# fused-sweep bring-up: forced parity tests, then A/B bench lines (fused vs single-level)
O=gpurun_out
mkdir -p $O
timeout 1200 env REXP_FUSE_FORCE=1 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_run_parity or lanes" 2>&1 | tail -15 > $O/f_tests_forced.txt
cat $O/f_tests_forced.txt
for c in c3_rsw_32x32_p16_x64 c1_rsw_16x16_p16; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline > $O/f_bench_${c%%_*}_fused.log 2>&1
  timeout 600 env REXP_FUSE_UP=0 REXP_FUSE_DOWN=0 python bench.py --config $c --steps 20 --no-cpu-baseline > $O/f_bench_${c%%_*}_single.log 2>&1
  timeout 600 env REXP_FUSE_FORCE=1 python bench.py --config $c --steps 20 --no-cpu-baseline > $O/f_bench_${c%%_*}_forced.log 2>&1
done
for f in $O/f_bench_*.log; do echo $f; tail -1 $f | python -c "
import sys, json
try:
    d = json.loads(sys.stdin.read())
    print(d['value'], d['ms_per_step'], d['impl_details']['merge_kernels'][-400:])
    print({k: v['ms_per_step'] for k, v in d['roofline']['per_class'].items()})
except Exception as e:
    print('ERR', e)
"; done
