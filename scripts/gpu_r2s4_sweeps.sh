# session-4: randomized parity sweeps against the oracle on the final build (bounded)
mkdir -p gpurun_out
timeout 420 python scripts/sweep_many.py 0 4000 > gpurun_out/sweep_many.log 2>&1; echo "many rc $? $(tail -1 gpurun_out/sweep_many.log)"
timeout 360 python scripts/sweep_wide.py 0 1200 > gpurun_out/sweep_wide.log 2>&1; echo "wide rc $? $(tail -1 gpurun_out/sweep_wide.log)"
timeout 240 python scripts/sweep_extra.py 300 > gpurun_out/sweep_extra.log 2>&1; echo "extra rc $? $(tail -1 gpurun_out/sweep_extra.log)"
