# A/B one kernel family by ncu launch times: LIBS="name:path ...", KREGEX=kernel regex, BENCH_ARGS
mkdir -p gpurun_out
for v in $LIBS; do name=${v%%:*}; lib=${v#*:}
COCLUST_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$KREGEX --csv --log-file gpurun_out/lk_$name.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 --graph off $BENCH_ARGS > /dev/null 2>&1
python - <<PY
import csv, io
lines = [l for l in open("gpurun_out/lk_$name.csv") if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]; vi = h.index("Metric Value")
t = [float(r[vi])/1e3 for r in rows[1:]]
print("$name", [round(x,1) for x in t[-${NLAST:-4}:]], "sum", round(sum(t[-${NLAST:-4}:]),1))
PY
done
