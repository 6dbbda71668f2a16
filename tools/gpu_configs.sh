# bench lines of the non-headline configurations with the final build
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc $?
for c in 5 6 7 1 2; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c rc $?; done
