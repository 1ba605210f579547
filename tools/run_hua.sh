# host-thread unit A (NEXT-1): parity tests, then C4/C3 bench lines with 0 / 8 / 14 host threads
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
for c in c4 c3; do
  for h in 8 14; do
    timeout 600 python bench.py --config $c --unit-a-host $h --no-cpu --e2e-runs 2 > gpurun_out/hua_${c}_h$h.log 2>&1
  done
done
