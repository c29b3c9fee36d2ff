# one ncu --set full capture of the fold-stage kernels of each workload (dram bytes per launch)
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none -k regex:"fold_f32" -s 2 -c 2 -o gpurun_out/tr_cfg3 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tr_cfg3.log 2>&1; echo cfg3 $?
for w in cfg4a cfg4b cfg4 cfg5; do
timeout 300 ncu --set full --clock-control none -k regex:"zero_i32|fold_pm1_tma|fold_finalize" -s 3 -c 3 -o gpurun_out/tr_$w python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tr_$w.log 2>&1; echo $w $?
done
