mkdir -p gpurun_out
bash scripts/gpu_ab_multi.sh "base orig" 2 --workload cfg5
bash scripts/gpu_ab_multi.sh "base orig" 1 --workload cfg4
for v in orig cur; do
C="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
if [ $v = cur ]; then unset TM_LIB_VARIANT; else export TM_LIB_VARIANT=$v; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tiled|match" -c 30 --csv --log-file gpurun_out/l_$v.csv $C > gpurun_out/ncu.log 2>&1; echo "ncu $v rc $?"
python scripts/show_launches.py gpurun_out/l_$v.csv 2>&1 | tail -3
done
unset TM_LIB_VARIANT
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 2>&1 | tail -9 | head -6
