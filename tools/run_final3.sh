# end of round 1, final state: GPU tests + smoke, C4 (default) and C3 bench lines
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/fin3_bench_c4.log 2>&1
timeout 900 python bench.py --config c3 > gpurun_out/fin3_bench_c3.log 2>&1
