# what paces deterministic mode: protocol off / fences off / full, rotated walk + slots (timing only)
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_relaxed.so timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_nowait.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/detprobe.txt
timeout 300 python exp/time_kernels.py c3 2>&1 | tee -a gpurun_out/detprobe.txt
