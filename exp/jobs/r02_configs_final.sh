# every bench config with the session's final build (3 timed steps each)
for c in c2 c4 c3_sparse c5_512k; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --skip-cpu > gpurun_out/r02z_bench_$c.json 2> gpurun_out/r02z_bench_$c.err
  head -c 200 gpurun_out/r02z_bench_$c.json; echo
done
