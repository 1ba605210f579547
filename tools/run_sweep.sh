timeout 900 python bench.py --no-cpu --unit-a-ctas 8 > gpurun_out/ua8_c4.log 2>&1
timeout 900 python bench.py --no-cpu --config c3 --unit-a-ctas 8 > gpurun_out/ua8_c3.log 2>&1
timeout 900 python bench.py --no-cpu --config c3 > gpurun_out/ua16_c3.log 2>&1
