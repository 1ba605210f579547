# tensor-core (3xTF32 mma.sync) Gram tiles of k_scd_pipe (W = 32, fast mode): parity, kernel time, C3 bench
timeout 600 python -m pytest tests/test_gpu_edge.py -m gpu -q -rf > gpurun_out/pytest_edge.log 2>&1; echo rc=$? >> gpurun_out/pytest_edge.log
DUHL_GRAM_TC=1 timeout 900 python -m pytest tests -m gpu -q -x -k "scd or solve or P7 or P8 or zero or fullsize" -rf > gpurun_out/pytest_tc.log 2>&1; echo rc=$? >> gpurun_out/pytest_tc.log
for tc in 0 1; do
  DUHL_GRAM_TC=$tc timeout 300 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 3 --ctas 139 > gpurun_out/prof_c3_tc$tc.log 2>&1
done
DUHL_GRAM_TC=1 timeout 900 python bench.py --config c3 --no-cpu > gpurun_out/bench_c3_tc1.log 2>&1
