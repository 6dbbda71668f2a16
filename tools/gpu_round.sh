set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench rc $?
cat gpurun_out/bench_c3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_list.log 2>&1; echo ncu list rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_oz -s 1 -c 1 -o gpurun_out/gram_oz_cfg3 python tools/prof_gram_oz.py 7 > gpurun_out/ncu_full.log 2>&1; echo ncu full rc $?
