# split deterministic backward: full GPU suite, sanitizers on the deterministic path, timing, bench line
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/dqf_gputest.log 2>&1; echo pytest_rc=$? >> gpurun_out/dqf_gputest.log
tail -3 gpurun_out/dqf_gputest.log
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_deterministic.py -m gpu -q -x > gpurun_out/dqf_memcheck.log 2>&1; tail -3 gpurun_out/dqf_memcheck.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_deterministic.py -m gpu -q -x -k "matches_default" > gpurun_out/dqf_racecheck.log 2>&1; tail -3 gpurun_out/dqf_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_deterministic.py -m gpu -q -x -k "matches_default" > gpurun_out/dqf_synccheck.log 2>&1; tail -3 gpurun_out/dqf_synccheck.log
for i in 1 2; do
  timeout 300 python exp/time_kernels.py c3 det
  BURST_LIB=exp/lib_prev.so timeout 300 python exp/time_kernels.py c3 det
done 2>&1 | grep -v Warn | tee gpurun_out/dqf_ab.txt
for L in "" exp/lib_prev.so; do
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c2 det
  BURST_LIB=$L timeout 300 python exp/time_kernels.py c3 causal det
done 2>&1 | grep -v Warn | tee -a gpurun_out/dqf_ab.txt
timeout 300 python exp/time_kernels.py c3 2>&1 | tee -a gpurun_out/dqf_ab.txt
timeout 600 python bench.py --deterministic --steps 5 --warmup 3 --skip-cpu > gpurun_out/dqf_bench_det.json 2> gpurun_out/dqf_bench_det.err
head -c 300 gpurun_out/dqf_bench_det.json
