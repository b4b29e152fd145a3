mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
CS_VARIANT=dbg CS_EXTRA_FLAGS="-DCS_ATTN_DEBUG" python -m paper_2603_18636_b200.build > gpurun_out/build2.log 2>&1 || { cat gpurun_out/build2.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "attn or fused or determinism" --timeout 120 --timeout-method thread -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error" | head -5
COCLUST_LIB=paper_2603_18636_b200/libcoclust_dbg.so timeout 300 python scripts/dbg_trace_v3.py
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms %.3f' % d['value'], d['stages_ms'], 'frac %.4f' % d['roofline']['frac'])"
