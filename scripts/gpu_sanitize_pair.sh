# compute-sanitizer over the CTA-pair assignment kernel (assign-step parity tests with K_s > 128)
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
K='assign_step and (500 or 300 or 1024) or exact_ties'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$K" -p no:cacheprovider > gpurun_out/san_${tool}_pair.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_${tool}_pair.log | tail -3
done
