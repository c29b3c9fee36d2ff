# session 3: cfg4 launch list + ncu full of its correlation kernels
mkdir -p gpurun_out
C="python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s3_launches_cfg4.csv $C > gpurun_out/s3_ncu4.log 2>&1; echo "ncu launches rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiled_prep|corr_tc_tiled" -s 2 -c 2 -o gpurun_out/s3_full_cfg4_corr $C > gpurun_out/s3_full4.log 2>&1; echo "ncu full rc $?"
