for env in "X=1" "TM_TILED_ACC=0" "TM_TILED_NCR=1" "TM_TILED_NCR=2" "TM_TILED_NT=64" "TM_TILED_NT=32"; do
  echo "== $env: $(env $env python scripts/dbg_seed.py 97 2>&1 | grep -A3 'rep 0 pair 1' | grep ' r[12] ' | tr '\n' ' ' | cut -c1-300)"
done
