timeout 900 python tools/round_trace.py c5 10 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csc.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "solve or adaptive or host or csc or virtual or fullsize or replay" 2>&1 | tail -1
timeout 900 python bench.py --config c5s --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c5s', l['ms_per_step'], l['value'], e['value'], e['time_to_eps_s'], e['rounds'])"
