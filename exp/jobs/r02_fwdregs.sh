# grid-masked forward: setmaxnreg split softmax/producer (208/88 default, 200/104, 192/120), c3_sparse
for i in 1 2; do
  for L in "" exp/lib_r200.so exp/lib_r192.so; do
    BURST_LIB=$L timeout 600 python bench.py --config c3_sparse --steps 3 --warmup 3 --skip-cpu 2>/dev/null | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); print(os.environ.get('BURST_LIB') or 'default', 'fwd', round(d['roofline']['lao_fwd']['ms_per_launch'],2), 'bwd', round(d['roofline']['ms_per_launch'],2), 'step', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
  done
done 2>&1 | tee gpurun_out/fwdregs.txt
