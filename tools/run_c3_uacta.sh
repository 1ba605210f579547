# C3 with fewer unit-A refresh CTAs beside the epoch (host threads take most of the refresh)
for u in 4 2; do
  timeout 600 python bench.py --config c3 --unit-a-ctas $u --no-cpu --e2e-runs 2 > gpurun_out/c3_ua$u.log 2>&1
done
