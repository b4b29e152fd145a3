# A/B variants of the attention kernel: full bench per variant
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  CS_VARIANT=$name CS_EXTRA_FLAGS="$flags" python -m paper_2603_18636_b200.build > gpurun_out/build_$name.log 2>&1 || { tail -5 gpurun_out/build_$name.log; continue; }
done
for v in base $VARIANTS; do
  name=${v%%:*}
  lib=paper_2603_18636_b200/libcoclust_$name.so; [ "$name" = base ] && lib=paper_2603_18636_b200/libcoclust.so
  COCLUST_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$name.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_$name.json')); print('$name', 'ms %.3f' % d['value'], 'attn %.3f' % d['stages_ms']['attention'], 'frac %.4f' % d['roofline']['frac'])"
done
