# final validation of HEAD: full GPU suite, smoke, default bench, deterministic bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02h_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_gputest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r02h_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r02h_smoke.log
timeout 600 python bench.py > gpurun_out/r02h_bench_c3.json 2> gpurun_out/r02h_bench_c3.err
timeout 600 python bench.py --deterministic --steps 5 --warmup 3 --skip-cpu > gpurun_out/r02h_bench_c3_det.json 2> gpurun_out/r02h_bench_c3_det.err
tail -3 gpurun_out/r02h_gputest.log; tail -2 gpurun_out/r02h_smoke.log; head -c 1500 gpurun_out/r02h_bench_c3.json; echo; head -c 400 gpurun_out/r02h_bench_c3_det.json
