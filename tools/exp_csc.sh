mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_csc.py tests/test_gpu_edge.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 900 python bench.py --config c5s > gpurun_out/csc_bench_c5s.json 2> gpurun_out/csc_bench_c5s.err
timeout 1500 python bench.py --config c5 > gpurun_out/csc_bench_c5.json 2> gpurun_out/csc_bench_c5.err
for c in c5s c5; do python -c "
import json; l=json.loads(open('gpurun_out/csc_bench_$c.json').read().strip().splitlines()[-1]); print('$c', l['ms_per_step'], l.get('gap_pass_GBps'), l['roofline']['frac'], (l.get('e2e') or {}).get('time_to_eps_s'))"; done
