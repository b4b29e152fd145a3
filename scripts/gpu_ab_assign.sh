mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "assign or kmeans or fused or determinism" --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for v in new old; do lib=paper_2603_18636_b200/libcoclust.so; [ $v = old ] && lib=paper_2603_18636_b200/libcoclust_old.so
COCLUST_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_assign --csv --log-file gpurun_out/la_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1
python - <<PY
import csv, io
lines = [l for l in open("gpurun_out/la_$v.csv") if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]; vi = h.index("Metric Value")
t = [float(r[vi])/1e3 for r in rows[1:]]
print("$v", [round(x,1) for x in t[-4:]])
PY
done
