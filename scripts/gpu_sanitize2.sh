# racecheck / initcheck over the smoke test (toy-size layer)
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python __graft_entry__.py > gpurun_out/san_racecheck_smoke.log 2>&1; echo "racecheck rc=$?"; tail -6 gpurun_out/san_racecheck_smoke.log
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python __graft_entry__.py > gpurun_out/san_initcheck_smoke.log 2>&1; echo "initcheck rc=$?"; tail -6 gpurun_out/san_initcheck_smoke.log
