# NEXT-3: offline profiler on synthetic Wan2.1-1.3B stacks -> schedule -> density-rule layer sweep
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python scripts/profile_schedule.py --config wan1.3b_480p --inputs 10 --out gpurun_out/schedule_wan13b.json; echo "profile rc=$?"
timeout 600 python scripts/sweep.py layers --config wan1.3b_480p --layers 30 --schedule gpurun_out/schedule_wan13b.json --out gpurun_out/sweep_layers_wan13b_sched.jsonl > gpurun_out/sweep_sched.log 2>&1; echo "sweep rc=$?"; tail -2 gpurun_out/sweep_sched.log
timeout 900 python scripts/profile_schedule.py --config wan14b_720p --inputs 2 --layers 4 --out gpurun_out/schedule_wan14b_4layers.json; echo "profile14 rc=$?"
