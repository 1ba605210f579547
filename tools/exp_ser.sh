mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kernel or 3" -p no:cacheprovider 2>&1 | tail -1
DUHL_SCD_TRACE=1 timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep "trace" | head -1
for v in "" tools/variants/libduhl_head.so; do
  echo "lib=$v"
  for rep in 1 2; do DUHL_LIB=$v timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"; done
  DUHL_LIB=$v timeout 300 python tools/prof_scd.py --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"
done
