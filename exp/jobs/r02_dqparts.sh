# lao_dq with 2 (default) or 4 dS warpgroups per tile: parity of both, timing vs HEAD
timeout 900 python -m pytest tests/test_gpu_deterministic.py tests/test_random_sweep.py tests/test_gpu_lao_level.py -m gpu -q -x > gpurun_out/dqp_tests.log 2>&1; echo rc=$? >> gpurun_out/dqp_tests.log; tail -2 gpurun_out/dqp_tests.log

for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det

  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/dqp_ab.txt
for L in "" exp/lib_prev.so; do
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c3 causal det
done 2>&1 | grep -v Warn | tee -a gpurun_out/dqp_ab.txt
