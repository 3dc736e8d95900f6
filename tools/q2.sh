# c3 launch list + ncu full capture of the merge GEMMs and leaf kernels of one c3 step
mkdir -p gpurun_out
R=q2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'k_cgemm|k_leaf_spec|k_upx|k_root' --launch-count 40 \
    -o gpurun_out/${R}_c3_full -f python tools/profile_step.py --config c3_rsw_32x32_p16_x64 > gpurun_out/${R}_ncu_full.log 2>&1
ls -la gpurun_out/ | tail
