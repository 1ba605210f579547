# round-2 experiments: hybrid staging share (C4), TPA cluster split with v0 in shared memory (C3)
export DUHL_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "solve_matches_oracle or virtual or unit_a" > gpurun_out/exp_pytest.txt 2>&1
tail -2 gpurun_out/exp_pytest.txt
B="python bench.py --steps 20 --warmup 5 --no-baselines --no-oracle-tte --e2e-runs 1 --no-cpu"
for sh in 0 0.2 0.3 0.45; do
  DUHL_STAGE_CE_SHARE=$sh timeout 600 $B > gpurun_out/exp_ce$sh.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/exp_ce$sh.json').read().splitlines()[-1]); p=l['pcie']
print('ce_share $sh', round(l['ms_per_step'],1), round(p['staging']['achieved_GBps'],1), round(p['achieved_GBps'],1), l['e2e']['time_to_eps_s'])"
done
timeout 900 python tools/tpa_vs_exact.py c3 128 > gpurun_out/exp_tpa_c1.log 2>&1; tail -1 gpurun_out/exp_tpa_c1.log
DUHL_TPA_CLUSTER=4 timeout 900 python tools/tpa_vs_exact.py c3 35 > gpurun_out/exp_tpa_c4.log 2>&1; tail -1 gpurun_out/exp_tpa_c4.log
DUHL_TPA_CLUSTER=2 timeout 900 python tools/tpa_vs_exact.py c3 70 > gpurun_out/exp_tpa_c2.log 2>&1; tail -1 gpurun_out/exp_tpa_c2.log
export DUHL_NO_HOST_OVERLAP=1
B3="python bench.py --steps 2 --warmup 6 --no-e2e --no-cpu --no-baselines --no-oracle-tte"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_c4.csv $B3 > gpurun_out/r02_ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_gather -c 1 -o gpurun_out/r02_stage_gather_c4 -f $B3 > gpurun_out/r02_ncu_gather.log 2>&1
tail -n 2 gpurun_out/r02_ncu_launch_c4.log gpurun_out/r02_ncu_gather.log
