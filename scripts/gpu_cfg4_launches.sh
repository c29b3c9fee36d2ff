mkdir -p gpurun_out
for w in cfg4a cfg4; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "$w rc $?"
done
