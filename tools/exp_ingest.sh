mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "host or pool or fullsize or c4 or c3" 2>&1 | tail -2
for sh in 0 0.5 0.6 0.7; do
  DUHL_INGEST_HOST_SHARE=$sh timeout 900 python bench.py --no-cpu --no-baselines --no-oracle-tte --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('share $sh', e['value'], e['create_s'], e['time_to_eps_s'])"
done
