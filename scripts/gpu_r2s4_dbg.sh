for env in "X=1" "TM_TILED_SPARSE=0" "TM_TILED_ACC=0" "TM_TILED_NCR=1" "TM_NO_PDL=1" "TM_CORR=ntt"; do
  echo "== $env: $(env $env python scripts/sweep_extra.py 60 2>&1 | tail -1) $(env $env python scripts/sweep_extra.py 60 2>&1 | grep -c FAIL)"
done
