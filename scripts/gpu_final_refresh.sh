# end-of-round refresh: every artifact profiles/r01 quotes, from one box
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 400 python bench.py > gpurun_out/bench_cfg2_final.json 2> gpurun_out/bench_cfg2_final.err; echo "cfg2 $(python scripts/show_bench.py gpurun_out/bench_cfg2_final.json | cut -c1-150)"
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc $?"
for w in cfg3 cfg4a cfg4b cfg4 cfg5; do
  timeout 400 python bench.py --workload $w > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-150)"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "ncu rc $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg3_final.csv python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "ncu cfg3 rc $?"
