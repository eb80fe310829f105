# dQ MMA in two chunk sets (drain starts on the chunks without dS^T under them): parity + A/B
timeout 900 python -m pytest tests/test_gpu_lao.py tests/test_gpu_properties.py tests/test_random_sweep.py tests/test_gpu_deterministic.py tests/test_gpu_large.py -m gpu -q -x > gpurun_out/dqsplit_tests.log 2>&1; echo rc=$? >> gpurun_out/dqsplit_tests.log
tail -3 gpurun_out/dqsplit_tests.log
for i in 1 2 3; do
  timeout 300 python exp/time_kernels.py c3
  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3
done 2>&1 | grep -v Warn | tee gpurun_out/dqsplit_ab.txt
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c2
  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c2
done 2>&1 | grep -v Warn | tee -a gpurun_out/dqsplit_ab.txt
timeout 300 python exp/time_kernels.py c3 causal 2>&1 | tee -a gpurun_out/dqsplit_ab.txt
BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 causal 2>&1 | tee -a gpurun_out/dqsplit_ab.txt
