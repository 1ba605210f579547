for rc in 16 1000000000; do
timeout 900 env DUHL_HEAVY_RUN_COLS=$rc python bench.py --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c4 runcols $rc', l['ms_per_step'], e['value'], e['time_to_eps_s'], e['time_to_eps_runs_s'], e['rounds'])"
done
