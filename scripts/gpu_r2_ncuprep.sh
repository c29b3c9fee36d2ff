mkdir -p gpurun_out
for w in cfg4 cfg5; do
C="python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiled_prep" -s 2 -c 1 -o gpurun_out/prep_$w $C > gpurun_out/ncu_prep_$w.log 2>&1; echo "ncu $w rc $?"
done
