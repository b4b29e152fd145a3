# NEXT-2 / NEXT-4 evidence: density-rule layer stacks with each selection variant / the k-means baseline
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for f in 0 1 2 3 256; do
  timeout 900 python scripts/sweep.py layers --config wan14b_720p --layers 40 --sel-flags $f --out gpurun_out/sweep_l14_f$f.jsonl > gpurun_out/sweep_l14_f$f.log 2>&1; echo "flags=$f rc=$?"; grep summary gpurun_out/sweep_l14_f$f.log
done
