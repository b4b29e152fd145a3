# A/B prebuilt libraries: LIBS="name:path ..." ; optional TESTS="pytest -k expr" run against the first lib.
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  first=${LIBS%% *}; COCLUST_LIB=${first#*:} timeout 900 python -m pytest tests/ -q -m gpu -x -k "$TESTS" --timeout 300 --timeout-method thread -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
fi
for round in 1 2; do
for v in $LIBS; do
  name=${v%%:*}; lib=${v#*:}
  COCLUST_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --reuse-steps 0 $BENCH_ARGS > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$name.json')); s=d['stages_ms']; print('$name', 'ms %.3f' % d['value'], 'attn %.3f' % s['attention'], 'clus %.3f' % s['cocluster'], 'sel %.3f' % s['select'], 'prep %.3f' % s['permute_v_worklist'], 'frac %.4f' % d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$name.err
done
done
