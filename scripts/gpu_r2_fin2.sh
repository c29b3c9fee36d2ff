for w in cfg4 cfg5 cfg4a; do bash scripts/gpu_ab_multi.sh "cur nofin nozero none" 1 --workload $w | cut -c1-110; done
