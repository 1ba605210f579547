# round-2 ncu evidence: launch lists of the C4 / C3 bench steps, --set full of the dominant kernels.
# ncu serialises kernels, so a pass-0 epoch that waits for staged columns could only time out:
# the profiled runs stage before the epoch (DUHL_NO_HOST_OVERLAP=1; same kernels, including the
# gather) -- their per-launch times, not the step overlap, are what these lists show.
set -x
export DUHL_NO_HOST_OVERLAP=1
B="python bench.py --steps 3 --warmup 5 --no-e2e --no-cpu --no-baselines --no-oracle-tte"
for c in c4 c3; do
  timeout 900 $B --config $c > gpurun_out/r02_small_$c.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches_$c.csv \
    $B --config $c > gpurun_out/r02_ncu_launch_$c.log 2>&1
done
timeout 300 python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/r02_p4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scd_gram -c 1 -o gpurun_out/r02_scd_gram_c4 -f \
  python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/r02_ncu_c4.log 2>&1
timeout 300 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --async_W 128 > gpurun_out/r02_p3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scd_tpa -c 1 -o gpurun_out/r02_scd_tpa_c3 -f \
  python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --async_W 128 > gpurun_out/r02_ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_stage_gather -s 2 -c 1 -o gpurun_out/r02_stage_gather_c4 -f \
  $B --config c4 > gpurun_out/r02_ncu_gather.log 2>&1
ls -la gpurun_out/*.ncu-rep
