timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for W in 12 8; do DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --passes 3 --W $W > gpurun_out/t4_$W.log 2>&1; done
for W in 32 24 16; do DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 3 --W $W > gpurun_out/t3_$W.log 2>&1; done
