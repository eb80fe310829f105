# full GPU suite (+ repeated grid-mask tests: flake check)
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_r02e.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02e.log
for i in $(seq 1 10); do timeout 300 python -m pytest tests/test_gpu_lao.py -m gpu -q -k "grid_mask or unaligned" 2>&1 | tail -1; done >> gpurun_out/pytest_r02e.log
tail -25 gpurun_out/pytest_r02e.log
