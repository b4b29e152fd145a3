# Round evidence: bench line, per-launch list, full ncu of the attention and assign kernels.
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsa_fwd -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu attn rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_assign|k_seg_mean|k_select_rows|k_permute_rows|k_csort_scatter|k_anchor_w|k_gamma|k_init_sample" -c 10 -o gpurun_out/prof_cluster python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu cluster rc=$?"
