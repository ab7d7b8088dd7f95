"""Summarise an ncu --set full capture of tc::kmatvec_tc_kernel into profiles/: the metric
subset bench.py and DESIGN.md cite (+ stall reasons per issue) and a warp-stall breakdown by
SASS instruction class (needs --import-source and -lineinfo).

  python tools/ncu_summary.py <report.ncu-rep> <metrics.json> <stalls.txt> <source command>
"""
import csv
import io
import json
import subprocess
import sys

rep, out_json, out_txt, src = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max", "sm__cycles_active.avg",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
d, units = {}, {}
for k in want:
    i = h.index(k)
    d[k] = v[i] if k in ("Kernel Name", "Grid Size", "Block Size") else float(v[i].replace(",", ""))
    units[k] = u[i]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
d["traffic_bytes_per_launch"] = sum(d[k] * scale[units[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
pre, post = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
d["stalls_per_issue"] = {k[len(pre):-len(post)]: float(v[i]) for i, k in enumerate(h)
                         if k.startswith(pre) and k.endswith(post)}
d["_source"] = src
d["_units"] = units
json.dump(d, open(out_json, "w"), indent=1)

srcp = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(srcp)))
hh = rows[1]
idx = {k: i for i, k in enumerate(hh)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
tot = sum(int(x[S] or 0) for x in data)
groups = {}
for i, x in enumerate(data):
    n = int(x[S] or 0)
    ins = x[1].strip()
    op = ins.split()[1] if ins.startswith("@") else (ins.split()[0] if ins else "")
    prev = data[i - 1][1] if i else ""
    if op.startswith("MUFU"):
        g = "MUFU.SQRT / MUFU.EX2 (kernel map on the SFU)"
    elif op == "BRA" and "TRYWAIT" in prev and "+0x8]" in prev and n > 0.05 * tot:
        g = "epilogue waiting for S(t) (s_full try-wait loop)"
    elif op == "BRA" and "TRYWAIT" in prev:
        g = "other mbarrier try-wait loops (producers, issuers, drains)"
    elif op.split(".")[0] in ("F2FP", "LOP3", "FADD2", "FFMA2", "FMUL2", "FADD", "FMUL", "FFMA"):
        g = "FP32 / ALU map + fp16 split (FFMA2, FMUL2, FADD2, LOP3, F2FP)"
    elif op.startswith("LDTM") or op.startswith("STTM"):
        g = "TMEM ld/st"
    elif op.startswith("UTCHMMA") or op.startswith("UTCBAR"):
        g = "MMA issue / commit"
    elif op.startswith("REDG") or op.startswith("STG"):
        g = "partial-sum drains (red.global / st.global)"
    else:
        g = "other (address, loop, predicate, barrier instructions)"
    groups[g] = groups.get(g, 0) + n
cols = ["stall_mio", "stall_long_sb", "stall_wait", "stall_not_selected", "stall_selected", "stall_short_sb",
        "stall_math", "stall_branch_resolving"]
with open(out_txt, "w") as f:
    f.write(f"{d['Kernel Name']}: warp-stall samples per SASS instruction (ncu --page source)\n")
    f.write(f"capture: {src}\ntotal samples {tot}\n\nshare of samples by instruction class:\n")
    for g, n in sorted(groups.items(), key=lambda t: -t[1]):
        f.write(f"  {100 * n / tot:5.1f}%  {g}\n")
    f.write("\ntop 25 instructions (stall reason counts):\n")
    for x in sorted(data, key=lambda x: -int(x[S] or 0))[:25]:
        n = int(x[S])
        f.write(f"  {100 * n / tot:5.1f}%  {x[1].strip()[:58]:58s} " +
                " ".join(f"{c[6:]}={x[idx[c]]}" for c in cols if x[idx[c]] not in ("0", "")) + "\n")
print(json.dumps({k: d[k] for k in ("gpu__time_duration.sum", "traffic_bytes_per_launch",
                                    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                                    "smsp__issue_active.avg.pct_of_peak_sustained_active",
                                    "launch__registers_per_thread")}))
