# round-2 GPU job: full GPU tests, C3 bench, reference arm
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_r02b.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02b.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3_r02b.json 2> gpurun_out/bench_c3_r02b.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02b.json 2>&1
tail -5 gpurun_out/pytest_r02b.log; head -c 4000 gpurun_out/bench_c3_r02b.json; tail -5 gpurun_out/bench_c3_r02b.err
