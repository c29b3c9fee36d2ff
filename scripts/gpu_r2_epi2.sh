for sp in 1 0; do echo "phases sparse=$sp"; TM_TILED_SPARSE=$sp timeout 300 python scripts/tiled_phases.py 16777216 16384 64 2>&1 | tail -9; done
