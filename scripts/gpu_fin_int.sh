mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_gpu_all.log)"
for w in cfg4a cfg4; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fold_finalize -c 6 --csv --log-file gpurun_out/fin_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo "$w finalize: $(python -c "
import csv
r=[x for x in csv.reader(open('gpurun_out/fin_$w.csv')) if len(x)>10]
h=r[0]; v=[float(x[h.index('Metric Value')].replace(',','')) for x in r[1:]]
print(round(sum(v)/len(v)/1000,1),'us')")"
done
