timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csc.py tests/test_gpu_tpa.py -m gpu -q -x -p no:cacheprovider -k "virtual or aggregat or gamma or linesearch or async or csc or tpa or cocoa or nccl" 2>&1 | tail -1
timeout 900 python bench.py --config c5s --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c5s', l['ms_per_step'], l['value'], e['value'], e['time_to_eps_s'], e['rounds'])"
timeout 900 python bench.py --config c3 --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('c3', l['ms_per_step'], l['value'], e['value'], e['time_to_eps_s'], e['rounds'])"
