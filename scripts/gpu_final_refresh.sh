# end-of-round refresh: every artifact profiles/r02 quotes, from one box
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $? $(tail -1 gpurun_out/smoke.log)"
timeout 600 python bench.py > gpurun_out/bench_cfg5_final.json 2> gpurun_out/bench_cfg5_final.err; echo "cfg5 $(python scripts/show_bench.py gpurun_out/bench_cfg5_final.json | cut -c1-170)"
for w in cfg2 cfg3 cfg4a cfg4b cfg4 cfg4c cfg4d t2 cfg1; do
  timeout 400 python bench.py --workload $w --no-cfg1 > gpurun_out/bench_${w}_final.json 2> gpurun_out/bench_${w}_final.err; echo "$w $(python scripts/show_bench.py gpurun_out/bench_${w}_final.json | cut -c1-170)"
done
for w in cfg5 cfg4 cfg3; do
  timeout 400 python bench.py --workload $w --pipeline 1 --no-cfg1 --no-cpu-baseline > gpurun_out/bench_${w}_onestream_final.json 2> gpurun_out/bench_${w}_onestream_final.err; echo "$w one stream $(python scripts/show_bench.py gpurun_out/bench_${w}_onestream_final.json | cut -c1-170)"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err; echo "ref rc $?"
timeout 600 python scripts/table1.py > gpurun_out/table1.json 2> gpurun_out/table1.err; echo "table1 rc $?"
timeout 600 python scripts/table2.py > gpurun_out/table2.json 2> gpurun_out/table2.err; echo "table2 rc $?"
C="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_final.csv $C > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
for w in cfg5 cfg4 cfg4b cfg4a; do
C="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"zero_i32|fold_pm1_tma|fold_finalize" -s 3 -c 3 -o gpurun_out/tr_$w $C > gpurun_out/tr_$w.log 2>&1; echo "ncu full $w rc $?"
done
C="python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiled_prep|corr_tc_tiled|tiled_reduce" -s 3 -c 3 -o gpurun_out/tr_cfg5_corr $C > gpurun_out/tr_cfg5_corr.log 2>&1; echo "ncu full cfg5 corr rc $?"
C="python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-cfg1"
$C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold_pm1_tma" -s 3 -c 1 -o gpurun_out/tr_cfg2 $C > gpurun_out/tr_cfg2.log 2>&1; echo "ncu full cfg2 rc $?"
# randomized parity sweeps against the oracle on the same build (bounded)
timeout 420 python scripts/sweep_many.py 0 4000 > gpurun_out/sweep_many.log 2>&1; echo "sweep many: $(tail -1 gpurun_out/sweep_many.log)"
timeout 400 python scripts/sweep_wide.py 0 1200 > gpurun_out/sweep_wide.log 2>&1; echo "sweep wide: $(tail -1 gpurun_out/sweep_wide.log)"
timeout 300 python scripts/sweep_extra.py 400 > gpurun_out/sweep_extra.log 2>&1; echo "sweep extra: $(tail -1 gpurun_out/sweep_extra.log)"
