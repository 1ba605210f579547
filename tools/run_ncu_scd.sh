# ncu --set full of the SCD kernel on the C3 / C4 shapes (one pass each)
python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c3 -f \
    python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 > gpurun_out/ncu_c3.log 2>&1
python tools/prof_scd.py --fast --passes 1 > gpurun_out/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c4 -f \
    python tools/prof_scd.py --fast --passes 1 > gpurun_out/ncu_c4.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lat tools/micro/lat.cu && /tmp/lat > gpurun_out/lat.log 2>&1
