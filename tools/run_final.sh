# end-of-round measurement set: GPU tests + smoke, bench lines (C4 default, C3, C4 GPU-only refresh,
# baselines), reference arm, ncu launch list of the default bench
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench_c4.log 2>&1
timeout 900 python bench.py --config c3 > gpurun_out/fin_bench_c3.log 2>&1
timeout 900 python bench.py --unit-a-host 0 --no-cpu > gpurun_out/fin_bench_c4_gpu_only.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin_b_small_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/fin_launches_c4.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin_ncu_launch_c4.log 2>&1
