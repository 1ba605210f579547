# passes-per-round sweep: the SCD epoch runs in the shadow of the PCIe-bound unit-A refresh
for p in 1 2 4; do timeout 900 python bench.py --no-cpu --passes $p > gpurun_out/sw_c4_p$p.log 2>&1; done
for p in 2 3; do timeout 900 python bench.py --no-cpu --config c3 --passes $p > gpurun_out/sw_c3_p$p.log 2>&1; done
