mkdir -p gpurun_out
TM_WS_POISON=1 timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_poison.log 2>&1; echo "poisoned suite: $(tail -1 gpurun_out/pytest_gpu_poison.log)"
grep -E "FAILED|ERROR" gpurun_out/pytest_gpu_poison.log | head -20
TM_WS_POISON=1 timeout 300 python scripts/sweep_many.py 0 1500 > gpurun_out/sweep_many_p.log 2>&1; echo "many poisoned rc $? $(tail -1 gpurun_out/sweep_many_p.log)"
TM_WS_POISON=1 timeout 300 python scripts/sweep_wide.py 0 500 > gpurun_out/sweep_wide_p.log 2>&1; echo "wide poisoned rc $? $(tail -1 gpurun_out/sweep_wide_p.log)"
TM_WS_POISON=1 timeout 200 python scripts/sweep_extra.py 200 > gpurun_out/sweep_extra_p.log 2>&1; echo "extra poisoned rc $? $(tail -1 gpurun_out/sweep_extra_p.log)"
