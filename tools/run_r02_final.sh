# round-2 final validation: GPU suite, smoke, the bench lines of every config, the reference arm.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.txt 2>&1
tail -3 gpurun_out/r02_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1
tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
for c in c3 c1 c2 c5s; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference_c4.json 2> gpurun_out/r02_bench_reference_c4.err
cat gpurun_out/r02_bench_*.json
