# iteration: build, attention parity tests, trace of one CTA, bench
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
CS_VARIANT=dbg CS_EXTRA_FLAGS="-DCS_ATTN_DEBUG" python -m paper_2603_18636_b200.build > gpurun_out/build2.log 2>&1 || { cat gpurun_out/build2.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "attn or fused or determinism or sampler" --timeout 120 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1; echo "pytest attn rc=$?"; tail -3 gpurun_out/pytest_attn.log
COCLUST_LIB=paper_2603_18636_b200/libcoclust_dbg.so timeout 300 python scripts/dbg_trace.py 2>&1 | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms', d['value'], 'stages', d['stages_ms'], 'frac', d['roofline']['frac'])"; tail -3 gpurun_out/bench.err
