python tools/prof_scd.py --fast --passes 1 --kernel 2 --ctas 140 > gpurun_out/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c4_pipe -f \
    python tools/prof_scd.py --fast --passes 1 --kernel 2 --ctas 140 > gpurun_out/ncu_c4.log 2>&1
