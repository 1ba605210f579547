# tensor-core Gram tiles at W < 32 (DUHL_GRAM_TC=2): fast-mode parity, C4-shaped kernel times
timeout 600 python -m pytest tests -m gpu -q -k "fast_mode" -rf > gpurun_out/pytest_fm.log 2>&1; echo rc=$? >> gpurun_out/pytest_fm.log
DUHL_GRAM_TC=2 timeout 600 python -m pytest tests -m gpu -q -k "fast_mode" -rf >> gpurun_out/pytest_fm.log 2>&1; echo rc=$? >> gpurun_out/pytest_fm.log
timeout 300 python tools/prof_scd.py --fast --passes 3 --kernel 1 --ctas 140 > gpurun_out/c4_k1.log 2>&1
for tc in 1 2; do
  DUHL_GRAM_TC=$tc timeout 300 python tools/prof_scd.py --fast --passes 3 --kernel 2 --ctas 140 > gpurun_out/c4_k2_tc$tc.log 2>&1
done
