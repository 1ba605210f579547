for e in "" "DUHL_NO_HEAVY_HOST_REFRESH=1"; do
env $e timeout 900 python bench.py --config c3 --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c3 [$e]', l['ms_per_step'], e['value'], e['time_to_eps_s'], e['time_to_eps_runs_s'], e['rounds'])"
done
timeout 900 python bench.py --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c4', l['ms_per_step'], e['value'], e['time_to_eps_s'], e['rounds'])"
