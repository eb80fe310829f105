# forward K/V stages 4 (default) vs 5, C3 and C2 and causal, interleaved
for i in 1 2 3; do
  timeout 300 python exp/time_kernels.py c3
  BURST_LIB=exp/lib_fs5.so timeout 300 python exp/time_kernels.py c3
done 2>&1 | grep -v Warn | tee gpurun_out/fwdstages.txt
for L in "" exp/lib_fs5.so; do
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c2
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c3 causal
done 2>&1 | grep -v Warn | tee -a gpurun_out/fwdstages.txt
