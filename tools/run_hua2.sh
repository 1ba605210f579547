# host-thread unit A: AVX-512 4-column dots; full-size parity; passes sweep with 14 host threads
python -m pytest tests -m gpu -x -q -k "unit_a_host or fullsize" > gpurun_out/pytest_gpu_hua.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_hua.log
for p in 1 2 3; do
  timeout 600 python bench.py --config c4 --unit-a-host 14 --passes $p --no-cpu --e2e-runs 2 > gpurun_out/hua2_c4_p$p.log 2>&1
done
for p in 2 3 4; do
  timeout 600 python bench.py --config c3 --unit-a-host 14 --passes $p --no-cpu --e2e-runs 2 > gpurun_out/hua2_c3_p$p.log 2>&1
done
