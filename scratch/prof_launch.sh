# per-kernel in-loop durations without ncu's cache flush, for the given libraries
for L in "$@"; do
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-c5"
BDEM_LIB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/launches_nc.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo "== $L"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_nc.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value')
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ki].split('(')[0]][r[mi]].append(float(r[vi].replace(',','')))
for k,m in agg.items():
    t=m['gpu__time_duration.sum']; print(k, len(t), round(sum(t)/len(t)/1e3,2), 'us', 'rd MB', round(sum(m['dram__bytes_read.sum'])/len(t)/1e6,1), 'wr MB', round(sum(m['dram__bytes_write.sum'])/len(t)/1e6,1))
PY
done
