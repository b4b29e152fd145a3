# A/B an environment switch: VAR=name, configs in CFGS ("args|args"), 3 alternating rounds
mkdir -p gpurun_out
IFS='|' read -ra CF <<< "${CFGS:---config wan14b_720p}"
for cfg in "${CF[@]}"; do
for round in 1 2 3; do
for v in 1 ""; do
  env $VAR=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --reuse-steps 0 $cfg > gpurun_out/abe.json 2>gpurun_out/abe.err
  python -c "
import json; d=json.load(open('gpurun_out/abe.json')); print('$cfg', '$VAR=[$v]', round(d['value'],3), round(d['stages_ms']['attention'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abe.err
done; done; done
