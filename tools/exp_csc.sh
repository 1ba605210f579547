mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_csc.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for v in "" tools/variants/libduhl_p768.so tools/variants/libduhl_p512.so; do
  for kb in 160 96; do
  echo "lib=$v kb=$kb"
  DUHL_LIB=$v DUHL_CSC_SMEM_KB=$kb timeout 600 python bench.py --config c5s --no-e2e --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l.get('gap_pass_GBps'))"
  done
done
DUHL_CSC_NO_PIPE=1 timeout 600 python bench.py --config c5s --no-e2e --no-cpu --no-baselines --no-oracle-tte 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nopipe', l['ms_per_step'], l.get('gap_pass_GBps'))"
