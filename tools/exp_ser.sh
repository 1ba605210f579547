mkdir -p gpurun_out
for v in tools/variants/libduhl_base.so tools/variants/libduhl_vupd1.so tools/variants/libduhl_vupd2.so tools/variants/libduhl_base.so; do
  echo "lib=$v"
  for rep in 1 2; do DUHL_LIB=$v timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep "^scd"; done
done
DUHL_LIB=tools/variants/libduhl_vupd2.so DUHL_SCD_TRACE=1 timeout 300 python tools/prof_scd.py --fast --passes 3 --ctas 140 --kernel 3 2>&1 | grep trace | head -1
