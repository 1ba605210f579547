mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ser_pytest_gpu.txt 2>&1
tail -3 gpurun_out/ser_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/ser_bench_c4.json 2> gpurun_out/ser_bench_c4.err
for c in c1 c2; do timeout 900 python bench.py --config $c > gpurun_out/ser_bench_$c.json 2> gpurun_out/ser_bench_$c.err; done
cat gpurun_out/ser_bench_c4.json
