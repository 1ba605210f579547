# end of round 1 (after the tensor-core Gram tiles): GPU tests + smoke, C3 bench line, C3 launch list,
# ncu --set full of the pipelined SCD kernel at the C3 bench shape
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --config c3 > gpurun_out/fin_bench_c3.log 2>&1
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin_b_small_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/fin_launches_c3.csv \
    python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin_ncu_launch_c3.log 2>&1
timeout 300 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --ctas 139 > gpurun_out/p3.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c3_tc -f \
  python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --ctas 139 > gpurun_out/ncu_c3.log 2>&1
