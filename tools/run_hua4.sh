# host unit A: certificate split + PCIe-aware share controller
python -m pytest tests -m gpu -x -q -k "unit_a_host or fullsize or solve" > gpurun_out/pytest_gpu_hua4.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_hua4.log
timeout 900 python bench.py --no-cpu --e2e-runs 2 > gpurun_out/hua4_c4.log 2>&1
timeout 900 python bench.py --config c3 --no-cpu --e2e-runs 2 > gpurun_out/hua4_c3.log 2>&1
