mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "host or pool" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu --no-baselines --no-oracle-tte --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c4', e['value'], e['create_s'], e['time_to_eps_s'], e['time_to_eps_runs_s'])"
timeout 600 python tools/solve_trace.py c4 2>&1 | tail -6
