# Secondary bench lines and density-rule stacks with the current build (one box, back to back)
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --config hunyuan_720p --no-cpu-baseline --no-e2e > gpurun_out/bench_hunyuan.json 2> gpurun_out/bench_hunyuan.err; echo "hunyuan rc=$?"
timeout 600 python bench.py --config wan1.3b_480p --no-cpu-baseline --no-e2e > gpurun_out/bench_wan13b.json 2> gpurun_out/bench_wan13b.err; echo "wan13b rc=$?"
timeout 600 python bench.py --sel-flags 256 --no-cpu-baseline --no-e2e > gpurun_out/bench_kmeans.json 2> gpurun_out/bench_kmeans.err; echo "kmeans rc=$?"
for f in 0 1; do
  timeout 900 python scripts/sweep.py layers --config wan14b_720p --layers 40 --sel-flags $f --out gpurun_out/sweep_l14_f$f.jsonl > gpurun_out/sweep_l14_f$f.log 2>&1; echo "flags=$f rc=$?"; grep summary gpurun_out/sweep_l14_f$f.log
done
timeout 900 python scripts/sweep.py layers --config wan1.3b_480p --layers 30 --out gpurun_out/sweep_l13.jsonl > gpurun_out/sweep_l13.log 2>&1; echo "l13 rc=$?"; grep summary gpurun_out/sweep_l13.log
for x in hunyuan wan13b kmeans; do python -c "
import json; d=json.load(open('gpurun_out/bench_$x.json')); s=d['stages_ms']; print('$x', 'ms %.3f' % d['value'], 'attn %.3f' % s['attention'], 'clus %.3f' % s['cocluster'], 'frac %.4f' % d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"; done
