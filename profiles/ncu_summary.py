import csv, subprocess, sys, json
rep, label = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
hdr, units, vals = r[0], r[1], r[2]
keys = ["Kernel Name","gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed","launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active","smsp__cycles_active.avg","sm__cycles_elapsed.avg",
        "launch__grid_size","launch__block_size","launch__shared_mem_per_block_dynamic",
        "lts__t_bytes.sum","smsp__inst_executed.sum","sm__cycles_elapsed.avg.per_second"]
res = {}
for k in keys:
    if k in hdr:
        i = hdr.index(k); res[k] = f"{vals[i]} {units[i]}".strip()
stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_",""): vals[i] for i,h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
res["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:8])
print(json.dumps({label: res}, indent=1))
