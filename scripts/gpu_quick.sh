# GPU tests + bench + launch list (no full ncu)
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/ -q -m gpu -x $PYTEST_ARGS --timeout 400 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --reuse-steps 0 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); s=d['stages_ms']; print('ms %.3f' % d['value'], s, 'frac %.4f' % d['roofline']['frac'], d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv 40 "" 2
