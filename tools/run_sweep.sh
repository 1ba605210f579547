for f in 0.1 0.06 0.15; do REFRESH=$f PASSES=2 timeout 600 python tools/solve_trace.py > gpurun_out/strace_c4_r$f.log 2>&1; done
