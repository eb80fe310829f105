# round-2 final job: GPU suite + smoke, driver-like C3 bench (K=20), reference arm,
# launch list and ncu metrics of the final build
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02f_smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02f_gputest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r02f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r02f_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02f_bench_c3_k20.json 2> gpurun_out/r02f_bench_c3_k20.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02f_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches_c3.csv python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/r02f_ncu_launch.log 2>&1
timeout 900 ncu --clock-control none -k regex:lao_ --csv --log-file gpurun_out/r02f_c3_metrics.csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed python tests/profile_step.py --config c3 --steps 1 > gpurun_out/r02f_ncu_metrics.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lao_bwd4 -c 1 -o gpurun_out/r02f_bwd_c2 python tests/profile_step.py --config c2 --steps 1 > gpurun_out/r02f_ncu_full.log 2>&1
tail -3 gpurun_out/r02f_gputest.log; cat gpurun_out/r02f_smoke.log | tail -2; head -c 2500 gpurun_out/r02f_bench_c3_k20.json; tail -3 gpurun_out/r02f_bench_c3_k20.err; head -c 800 gpurun_out/r02f_bench_ref.json; tail -2 gpurun_out/r02f_ncu_metrics.log gpurun_out/r02f_ncu_full.log
