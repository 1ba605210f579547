mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/prefill_pytest.txt 2>&1; tail -2 gpurun_out/prefill_pytest.txt
timeout 900 python bench.py --no-cpu --no-baselines --no-oracle-tte > gpurun_out/prefill_c4.json 2> gpurun_out/prefill_c4.err
DUHL_NO_PREFILL=1 timeout 900 python bench.py --no-cpu --no-baselines --no-oracle-tte > gpurun_out/noprefill_c4.json 2> gpurun_out/noprefill_c4.err
for f in prefill_c4 noprefill_c4; do python -c "
import json; l=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); e=l['e2e']; print('$f', l['ms_per_step'], e['value'], e['time_to_eps_s'], e['time_to_eps_runs_s'], e['create_s'], e['rounds'], e['h2d_bytes_per_step'], e['state_check'])"; done
