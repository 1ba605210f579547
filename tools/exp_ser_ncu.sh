mkdir -p gpurun_out
timeout 300 python tools/prof_scd.py --fast --passes 1 --ctas 140 --kernel 3 > gpurun_out/ser_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scd_ser -c 1 -o gpurun_out/ser_c4 -f \
  python tools/prof_scd.py --fast --passes 1 --ctas 140 --kernel 3 > gpurun_out/ser_ncu.log 2>&1
tail -3 gpurun_out/ser_ncu.log
