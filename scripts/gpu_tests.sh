# Build + the GPU test suite (all of it, or $PYTEST_ARGS) + the racecheck microtest of the CTA-pair alloc.
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests/ -q -m gpu ${PYTEST_ARGS} --timeout 900 --timeout-method thread -p no:cacheprovider -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; grep -E "passed|failed|PASSED.*midsize|^FAILED|Error" gpurun_out/pytest_gpu.log | tail -25
if [ -n "$RACE" ]; then
  (cd scripts/micro && ./pair_alloc_race && compute-sanitizer --tool racecheck ./pair_alloc_race > ../../gpurun_out/race_alloc.log 2>&1; compute-sanitizer --tool racecheck ./pair_alloc_race presync > ../../gpurun_out/race_alloc_presync.log 2>&1); tail -3 gpurun_out/race_alloc.log gpurun_out/race_alloc_presync.log
fi
