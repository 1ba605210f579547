# round-1 measurement set: bench lines (C4 default, C3), reference arm, launch lists, ncu of the C4 SCD kernel at the bench shape
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config c3 > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_small_$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 300 python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/p4.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c4_final -f \
  python tools/prof_scd.py --fast --passes 1 --ctas 140 > gpurun_out/ncu_c4.log 2>&1
timeout 300 python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --ctas 139 > gpurun_out/p3.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scd -c 1 -o gpurun_out/scd_c3_final -f \
  python tools/prof_scd.py --fast --lasso --d 40000 --n 50176 --passes 1 --ctas 139 > gpurun_out/ncu_c3.log 2>&1
