timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 3 --ctas 139 > gpurun_out/t3_g4.log 2>&1
