# bench lines for configs 3 (headline), 2, 1, 5 + the config-3 launch list + ncu --set full of
# the Ozaki kernels (each only after its command exited 0 without ncu)
set -x
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3 rc $?
for c in 2 1; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c rc $?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo ncu list rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_oz -s 1 -c 1 -o gpurun_out/gram_oz_cfg3 -f python tools/prof_gram_oz.py 7 > gpurun_out/ncu_full.log 2>&1; echo ncu gram rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 2 -c 1 -o gpurun_out/oz_gemm_ls_cfg3 -f python tools/prof_ls.py > gpurun_out/ncu_gemm.log 2>&1; echo ncu gemm rc $?
