for cl in 1 0; do echo "cl=$cl"; TM_TILED_CL=$cl timeout 300 python scripts/tiled_phases.py 2147483648 65536 1 2>&1 | tail -8; done
