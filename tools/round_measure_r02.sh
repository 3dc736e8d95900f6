#!/bin/bash
# Round-2 GPU call: the full GPU parity suite, the bench lines kept under
# profiles/ (c3 headline, c1, c2r, the c2 / c4 shards, the reference arm), the
# ncu launch lists (time + DRAM bytes of every launch of the bench's timed
# region) and an ncu --set full capture of the top kernels of a c3 step
# (exported to CSV on the box; the .ncu-rep stays in /tmp).
set -u
R=${1:-r02}
O=gpurun_out
mkdir -p $O
STAGE=${STAGE:-all}
if [ "$STAGE" = all ] || [ "$STAGE" = tests ]; then
  timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > $O/${R}_gpu_tests.txt
fi
if [ "$STAGE" = all ] || [ "$STAGE" = bench ]; then
  timeout 600 python bench.py > $O/${R}_bench_c3.log 2>&1
  timeout 300 python bench.py --config c1_rsw_16x16_p16 --no-cpu-baseline > $O/${R}_bench_c1.log 2>&1
  timeout 300 python bench.py --config c2r_wave_8x8_p16 --steps 20 --no-cpu-baseline > $O/${R}_bench_c2r.log 2>&1
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_bench_reference.log 2>&1
fi
if [ "$STAGE" = all ] || [ "$STAGE" = shards ]; then
  timeout 1200 python bench.py --config c2_wave_32x32_p16 --shard auto --steps 5 --no-cpu-baseline > $O/${R}_bench_c2_shard.log 2>&1
  timeout 1500 python bench.py --config c4_wave_64x64_p12 --shard auto --steps 5 --no-cpu-baseline > $O/${R}_bench_c4_shard.log 2>&1
fi
if [ "$STAGE" = all ] || [ "$STAGE" = ncu ]; then
  M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
  for c in c3_rsw_32x32_p16_x64 c1_rsw_16x16_p16; do
    timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
        --log-file $O/${R}_launches_${c%%_*}.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline \
        > $O/${R}_ncu_launch_${c%%_*}.log 2>&1
  done
  timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:'k_cgemm|k_leaf_gemm|k_upx|k_root|k_spec|k_recover' --launch-count 40 \
      -o /tmp/${R}_c3_full -f python tools/profile_step.py --config c3_rsw_32x32_p16_x64 > $O/${R}_ncu_full.log 2>&1
  ncu -i /tmp/${R}_c3_full.ncu-rep --page raw --csv > $O/${R}_c3_raw.csv 2>/dev/null
fi
cat $O/${R}_gpu_tests.txt 2>/dev/null
for f in c3 c1 c2r reference c2_shard c4_shard; do [ -f $O/${R}_bench_$f.log ] && tail -1 $O/${R}_bench_$f.log | cut -c1-200; done
ls -la $O | tail -30
