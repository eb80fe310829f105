# deterministic dQ with the paired backward: parity + A/B vs the unpaired ordered kernel
timeout 600 python -m pytest tests/test_gpu_deterministic.py tests/test_random_sweep.py -m gpu -q -x > gpurun_out/detpair_tests.log 2>&1; echo rc=$? >> gpurun_out/detpair_tests.log
tail -3 gpurun_out/detpair_tests.log
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_detold.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/detpair_ab.txt
timeout 300 python exp/time_kernels.py c3 2>&1 | tee -a gpurun_out/detpair_ab.txt
timeout 300 python exp/time_kernels.py c3 causal det 2>&1 | tee -a gpurun_out/detpair_ab.txt
BURST_LIB=exp/lib_detold.so timeout 300 python exp/time_kernels.py c3 causal det 2>&1 | tee -a gpurun_out/detpair_ab.txt
timeout 600 python bench.py --deterministic --steps 5 --warmup 3 --skip-cpu > gpurun_out/detpair_bench.json 2> gpurun_out/detpair_bench.err
head -c 600 gpurun_out/detpair_bench.json
