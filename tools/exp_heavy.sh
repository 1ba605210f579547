timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "heavy or budget or fullsize or c3 or c4 or solve or host" > gpurun_out/heavy_pytest.txt 2>&1; tail -1 gpurun_out/heavy_pytest.txt
timeout 1500 python tools/sweep_c4.py --config c3 0.1:3 0.1:4 0.1:5 0.12:4 0.08:4 > gpurun_out/sweep_c3c.log 2>&1; cat gpurun_out/sweep_c3c.log | grep '^{'
timeout 900 python bench.py --config c3 --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c3', l['ms_per_step'], e['value'], e['time_to_eps_s'], e['time_to_eps_runs_s'], e['rounds'])"
