# session 3: per-CTA phase timeline of corr_tc_tiled at cfg5 and cfg4
mkdir -p gpurun_out
timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 > gpurun_out/s3_ph_cfg5.txt 2>&1; echo "cfg5 rc $?"; cat gpurun_out/s3_ph_cfg5.txt
TM_TILED_NT=64 timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 > gpurun_out/s3_ph_cfg5_nt64.txt 2>&1; echo "cfg5 nt64 rc $?"; cat gpurun_out/s3_ph_cfg5_nt64.txt
timeout 300 python scripts/tiled_phases.py 16777216 16384 64 > gpurun_out/s3_ph_cfg4.txt 2>&1; echo "cfg4 rc $?"; cat gpurun_out/s3_ph_cfg4.txt
