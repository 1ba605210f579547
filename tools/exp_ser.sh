for v in tools/variants/libduhl_base.so tools/variants/libduhl_arrive.so tools/variants/libduhl_base.so tools/variants/libduhl_arrive.so; do
  echo "lib=$v"
  for rep in 1 2; do DUHL_LIB=$v timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"; done
done
DUHL_LIB=tools/variants/libduhl_arrive.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "kernel or ser or 3 or solve" 2>&1 | tail -1
