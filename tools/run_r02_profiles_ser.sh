# round-2 ncu evidence after k_scd_ser: the C4 bench step launch list and --set full of k_scd_ser.
# (DUHL_NO_HOST_OVERLAP=1: ncu serialises kernels, see run_r02_profiles.sh)
set -x
export DUHL_NO_HOST_OVERLAP=1
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 5 --no-e2e --no-cpu --no-baselines --no-oracle-tte"
timeout 900 $B --config c4 > gpurun_out/r02s_small_c4.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02s_launches_c4.csv \
  $B --config c4 > gpurun_out/r02s_ncu_launch_c4.log 2>&1
timeout 300 python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/r02s_p4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scd_ser -c 1 -o gpurun_out/r02s_scd_ser_c4 -f \
  python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/r02s_ncu_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r02s_launches_c4.csv
