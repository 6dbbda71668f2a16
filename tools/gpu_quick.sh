# quick GPU check: the GPU test suite + the default bench line
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])
print({k: round(v,3) for k,v in d['stages_ms_per_step'].items()})"
