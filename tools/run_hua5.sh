# host unit A: share up to 1; staging copies overlapped with the epoch when the host takes the refresh
python -m pytest tests -m gpu -x -q -k "unit_a_host" > gpurun_out/pytest_gpu_hua5.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_hua5.log
DUHL_HOST_OVERLAP=1 python -m pytest tests -m gpu -x -q -k "unit_a_host" >> gpurun_out/pytest_gpu_hua5.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_hua5.log
timeout 900 python bench.py --no-cpu --e2e-runs 2 > gpurun_out/hua5_c4.log 2>&1
DUHL_HOST_OVERLAP=1 timeout 900 python bench.py --no-cpu --e2e-runs 2 > gpurun_out/hua5_c4_ov.log 2>&1
DUHL_HOST_OVERLAP=1 timeout 900 python bench.py --config c3 --no-cpu --e2e-runs 2 > gpurun_out/hua5_c3_ov.log 2>&1
