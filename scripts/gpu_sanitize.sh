# compute-sanitizer over the smoke test and small parity tests (memcheck, synccheck)
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py > gpurun_out/san_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -4 gpurun_out/san_memcheck_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "tiny or split_kv or toy or variants_bitexact and 16 or kmeans_assign_step and 2048 or permute_bitexact and 5000" -p no:cacheprovider > gpurun_out/san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -6 gpurun_out/san_memcheck_tests.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python __graft_entry__.py > gpurun_out/san_synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?"; tail -4 gpurun_out/san_synccheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_profile.py -q -x -m gpu -k "uniform" -p no:cacheprovider > gpurun_out/san_memcheck_profile.log 2>&1; echo "memcheck profile rc=$?"; tail -4 gpurun_out/san_memcheck_profile.log
