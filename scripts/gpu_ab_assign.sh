# A/B the assignment GEMM: tests on the first lib, ncu launch times of k_assign per lib (LIBS="name:path ...")
mkdir -p gpurun_out
first=${LIBS%% *}; COCLUST_LIB=${first#*:} timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "assign or kmeans or fused or determinism" --timeout 300 -p no:cacheprovider 2>&1 | tail -1
for v in $LIBS; do name=${v%%:*}; lib=${v#*:}
COCLUST_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_assign --csv --log-file gpurun_out/la_$name.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1
python - <<PY
import csv, io
lines = [l for l in open("gpurun_out/la_$name.csv") if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]; vi = h.index("Metric Value")
t = [float(r[vi])/1e3 for r in rows[1:]]
print("$name", [round(x,1) for x in t[-4:]])
PY
done
