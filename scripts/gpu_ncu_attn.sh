# full ncu capture (with source) of one attention launch
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsa_fwd -c 1 -f -o gpurun_out/prof_attn${TAG} python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_attn.log 2>&1; echo "ncu attn rc=$?"
tail -3 gpurun_out/ncu_attn.log
