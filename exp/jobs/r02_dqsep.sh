# deterministic mode = lao_bwd4 (dK/dV only) + query-stationary lao_dq: parity, then timing vs the ordered chain
timeout 900 python -m pytest tests/test_gpu_deterministic.py tests/test_random_sweep.py tests/test_gpu_lao_level.py -m gpu -q -x > gpurun_out/dqsep_tests.log 2>&1; echo rc=$? >> gpurun_out/dqsep_tests.log
tail -25 gpurun_out/dqsep_tests.log
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/dqsep_ab.txt
for L in "" exp/lib_prev.so; do
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c2 det
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c3 causal det
done 2>&1 | grep -v Warn | tee -a gpurun_out/dqsep_ab.txt
