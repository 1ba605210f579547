timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_ce.log 2>&1
DUHL_ZERO_COPY_GAPS=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_zc.log 2>&1
