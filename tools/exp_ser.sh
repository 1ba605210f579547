mkdir -p gpurun_out
for v in "" tools/variants/libduhl_w12.so tools/variants/libduhl_w16.so; do
  echo "lib=$v"
  DUHL_LIB=$v timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"
  DUHL_LIB=$v timeout 300 python tools/prof_scd.py --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"
done
DUHL_LIB=tools/variants/libduhl_w12.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kernel or 3" -p no:cacheprovider 2>&1 | tail -2
