# randomized parity sweeps against the oracle (DESIGN 8b) on the current build
mkdir -p gpurun_out
timeout 1200 python scripts/sweep_many.py 0 10000 > gpurun_out/sweep_many.log 2>&1; echo "many rc $? $(tail -1 gpurun_out/sweep_many.log)"
timeout 900 python scripts/sweep_wide.py 0 3500 > gpurun_out/sweep_wide.log 2>&1; echo "wide rc $? $(tail -1 gpurun_out/sweep_wide.log)"
timeout 600 python scripts/sweep_extra.py 1000 > gpurun_out/sweep_extra.log 2>&1; echo "extra rc $? $(tail -1 gpurun_out/sweep_extra.log)"
