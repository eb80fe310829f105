# deterministic dQ with rotated walks and per-(epoch, member) chains into separate slots
timeout 900 python -m pytest tests/test_gpu_deterministic.py tests/test_random_sweep.py tests/test_gpu_lao.py tests/test_gpu_lao_level.py -m gpu -q -x > gpurun_out/detrot_tests.log 2>&1; echo rc=$? >> gpurun_out/detrot_tests.log
tail -5 gpurun_out/detrot_tests.log
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/detrot_ab.txt
timeout 300 python exp/time_kernels.py c3 causal det 2>&1 | tee -a gpurun_out/detrot_ab.txt
timeout 300 python exp/time_kernels.py c2 det 2>&1 | tee -a gpurun_out/detrot_ab.txt
timeout 300 python exp/time_kernels.py c3 2>&1 | tee -a gpurun_out/detrot_ab.txt
BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 2>&1 | tee -a gpurun_out/detrot_ab.txt
