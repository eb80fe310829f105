# round-2 GPU job: GPU tests, smoke, C3 bench, reference arm, ncu launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/pytest_r02c.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02c.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r02c.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3_r02c.json 2> gpurun_out/bench_c3_r02c.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02c.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/ncu_launch.log 2>&1
tail -5 gpurun_out/pytest_r02c.log; cat gpurun_out/smoke_r02c.log; head -c 3000 gpurun_out/bench_c3_r02c.json; tail -3 gpurun_out/bench_c3_r02c.err; head -c 1500 gpurun_out/bench_ref_r02c.json
