timeout 900 python -m pytest tests -m gpu -x -q -k "scd or P7 or P8 or zero or solve" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 3 --ctas 139 > gpurun_out/t3_32.log 2>&1
DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --passes 3 --kernel 2 --ctas 140 > gpurun_out/t4_pipe.log 2>&1
DUHL_SCD_TRACE=1 timeout 120 python tools/prof_scd.py --fast --passes 3 --kernel 1 --ctas 140 > gpurun_out/t4_gram.log 2>&1
