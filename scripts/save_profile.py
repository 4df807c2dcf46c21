"""Copy one GPU session's evidence from gpurun_out/ into profiles/<round tag>/:
bench line, per-pass detail, ncu launch list, ncu --set full summary of the
pass kernels, and profiles/ncu_traffic.json (DRAM bytes per k_pass16 launch,
read by bench.py as roofline.traffic).

    python scripts/save_profile.py v3 r01_v3
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, dest = sys.argv[1], sys.argv[2]
src = os.path.join(ROOT, "gpurun_out")
out = os.path.join(ROOT, "profiles", dest)
os.makedirs(out, exist_ok=True)
for name, new in ((f"bench_{tag}.log", "bench.json"), (f"pass_{tag}.log", "passes.txt"),
                  (f"launches_{tag}.csv", "launches.csv"), (f"pytest_gpu_{tag}.log", "pytest_gpu.txt")):
    if os.path.exists(os.path.join(src, name)):
        shutil.copy(os.path.join(src, name), os.path.join(out, new))
rep = os.path.join(src, f"prof_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "sm__cycles_elapsed.avg.per_second"]
    launches = []
    with open(os.path.join(out, "ncu_full_summary.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, k_pass16 launches of one LABS n=26 p=10 step ({rep})\n")
        for r in rows[2:]:
            f.write("-" * 70 + "\n")
            d = {}
            for k in keep:
                if k in hdr:
                    i = hdr.index(k)
                    f.write(f"{k:75s} {r[i]} {units[i]}\n")
                    d[k] = (r[i], units[i])
            def gb(k):
                v, u = d[k]
                return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]
            launches.append({"kernel": d["Kernel Name"][0], "dram_bytes": gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"),
                             "us": float(d["gpu__time_duration.sum"][0])})
    tr = {"n": 26, "source": f"profiles/{dest}/ncu_full_summary.txt", "launches": launches,
          "dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) / max(1, len(launches))}
    tfile = os.path.join(src, f"traffic_{tag}.csv")
    if os.path.exists(tfile):  # every pass of one step: traffic per launch comparable to bench's algorithmic bytes
        shutil.copy(tfile, os.path.join(out, "traffic_step.csv"))
        rows = [r for r in csv.reader(open(tfile)) if len(r) > 10]
        h = rows[0]
        ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        ids = {}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[1:]:
            if r[mi].startswith("dram__bytes"):
                ids.setdefault(r[0], [r[ki], 0.0])[1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        if ids:
            tot = sum(v[1] for v in ids.values())
            tr.update({"dram_bytes_per_launch": tot / len(ids), "step_launches": len(ids), "step_dram_bytes": tot,
                       "source": f"profiles/{dest}/traffic_step.csv (all k_pass16 launches of one step)"})
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(tr, f, indent=1)
    print(json.dumps(tr, indent=1))
