for u in 0 4 6; do
  timeout 900 python bench.py --unit-a-ctas $u --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('uactas $u', l['ms_per_step'], l['roofline']['frac'], l['config']['scd_kernel'], (l['pcie'] or {}).get('staging',{}).get('achieved_GBps'), e['time_to_eps_s'])"
done
