# One GPU session: build, all GPU tests, smoke, bench, ncu launch list, full ncu of the attention
# kernel and of the assignment GEMM.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
[ -n "$SKIP_TESTS" ] || { timeout 1500 python -m pytest tests/ -q -m gpu --timeout 400 --timeout-method thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu.log; }
timeout 900 python bench.py --steps 10 --warmup 3 --reuse-steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; tail -c 400 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
[ -n "$SKIP_FULL" ] || { timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsa_fwd -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1; echo "ncu attn rc=$?"; }
[ -n "$SKIP_FULL" ] || { timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assign -c 2 -o gpurun_out/prof_assign python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --reuse-steps 0 > /dev/null 2>&1; echo "ncu assign rc=$?"; }
