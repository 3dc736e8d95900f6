#!/bin/bash
# One GPU call: parity suite, the bench lines kept under profiles/, the ncu
# launch list of the bench's timed region and one full capture of the two
# spectral leaf kernels (each ncu pass only after its command exited 0).
set -u
R=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/${R}_gpu_tests.txt
python bench.py > $O/${R}_bench_c1.log 2>&1
python bench.py --config c3_rsw_32x32_p16_x64 --steps 5 --warmup 3 --no-cpu-baseline > $O/${R}_bench_c3.log 2>&1
python bench.py --config c2r_wave_8x8_p16 --steps 20 --warmup 3 --no-cpu-baseline > $O/${R}_bench_c2r.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_bench_reference.log 2>&1
if python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${R}_pre_ncu.log 2>&1; then
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${R}_ncu_launch.log 2>&1
fi
if python tools/profile_step.py > $O/${R}_ps.log 2>&1; then
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_leaf_spec \
      -o $O/${R}_leaf_full -f python tools/profile_step.py > $O/${R}_ncu_full.log 2>&1
fi
if [ -s $O/${R}_ps.log ]; then
  ncu --profile-from-start off --set full --clock-control none -k regex:'k_cgemm|k_gemv_sym' --launch-count 24 \
      -o $O/${R}_merge_full -f python tools/profile_step.py > $O/${R}_ncu_merge.log 2>&1 &&
  ncu -i $O/${R}_merge_full.ncu-rep --page raw --csv > $O/${R}_merge_raw.csv && rm -f $O/${R}_merge_full.ncu-rep
fi
cat $O/${R}_gpu_tests.txt
for f in c1 c3 c2r reference; do tail -1 $O/${R}_bench_$f.log | cut -c1-300; done
