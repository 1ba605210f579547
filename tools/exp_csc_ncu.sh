mkdir -p gpurun_out
B="python bench.py --config c5s --steps 2 --warmup 3 --no-e2e --no-cpu --no-baselines --no-oracle-tte"
timeout 600 $B > gpurun_out/csc_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csc_scd -s 3 -c 1 -o gpurun_out/csc_scd -f $B > gpurun_out/csc_scd_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c5s.csv $B > gpurun_out/csc_launch.log 2>&1
tail -2 gpurun_out/csc_scd_ncu.log
