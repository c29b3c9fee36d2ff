mkdir -p gpurun_out
for w in cfg4 cfg4a; do
C="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold_pm1_tma|fold_finalize|zero_i32" -s 6 -c 3 -o gpurun_out/prof_fold_$w $C > gpurun_out/ncu_$w.log 2>&1; echo "ncu $w rc $?"
done
bash scripts/gpu_ab_multi.sh "base nocomp" 1 --workload cfg4
