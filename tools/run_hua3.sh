# host-thread unit A at C4 (2 passes): AVX-512 4-column dots vs AVX2 single, balanced vs fixed share
for v in 512 2; do
  for sh in -1 0.7; do
    if [ $v = 2 ]; then export DUHL_HOST_NO_AVX512=1; else unset DUHL_HOST_NO_AVX512; fi
    timeout 600 python bench.py --config c4 --unit-a-host 14 --host-share $sh --no-cpu --e2e-runs 1 > gpurun_out/hua3_v${v}_s$sh.log 2>&1
  done
done
