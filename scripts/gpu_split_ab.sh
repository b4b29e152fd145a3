mkdir -p gpurun_out
LIBS="new:paper_2603_18636_b200/libcoclust.so old:paper_2603_18636_b200/libcoclust_old.so" TESTS="attn or fused or smoke or determinism or fullsize" bash scripts/gpu_ab.sh
for kc in "--kq 256 --kk 1024" "--kq 1024 --kk 1024"; do for v in new old; do lib=paper_2603_18636_b200/libcoclust.so; [ $v = old ] && lib=paper_2603_18636_b200/libcoclust_old.so
COCLUST_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --reuse-steps 0 $kc > gpurun_out/k_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/k_$v.json')); s=d['stages_ms']; print('$v $kc', 'ms %.3f' % d['value'], 'attn %.3f' % s['attention'], 'frac %.4f' % d['roofline']['frac'])"; done; done
