timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csc.py -m gpu -q -x -p no:cacheprovider -k "solve or adaptive or host or csc or virtual or replay" 2>&1 | tail -1
timeout 300 python tools/create_timing.py c1 6 solve 2>&1 | tail -6
for c in c1 c5s; do
timeout 900 python bench.py --config $c --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('$c', l['ms_per_step'], l['value'], e['value'], e['time_to_eps_s'], e['create_plus_solve_runs_s'])"
done
