# multi-GPU code paths on one device: tests, torchrun x1 with Ulysses and head-parallel
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_dist.py -q -m gpu --timeout 200 -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error" | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --config hunyuan_720p --parallel ulysses --no-cpu-baseline > gpurun_out/bench_uly.json 2> gpurun_out/bench_uly.err; echo "uly rc=$?"; cut -c1-600 gpurun_out/bench_uly.json; tail -3 gpurun_out/bench_uly.err


