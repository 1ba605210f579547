# C3 passes per round after the tensor-core Gram tiles (host unit A, bench defaults otherwise)
for p in 2 4; do
  timeout 600 python bench.py --config c3 --passes $p --no-cpu --e2e-runs 2 > gpurun_out/c3_p$p.log 2>&1
done
