# end-of-round check: smoke, the GPU suite, the default bench line and the reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc $?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
cat gpurun_out/bench_ref.json
