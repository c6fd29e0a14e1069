"""Summarise ncu reports in gpurun_out/ into profiles/ (run here, no GPU): per kernel launch the
duration, DRAM bytes, throughput %, instructions, registers, occupancy and top stall reasons."""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed_op_shfl.sum" ]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3,
        "us": 1.0, "ms": 1e3, "ns": 1e-3}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:160]}
        for key in KEYS:
            if key in d and d[key] not in ("", "n/a"):
                v = float(d[key].replace(",", ""))
                k[key] = v * UNIT.get(u.get(key, ""), 1.0) if u.get(key, "") in UNIT else v
                if u.get(key):
                    k[key + ".unit"] = "byte" if "byte" in u[key] else ("us" if u[key] in ("usecond", "msecond", "nsecond", "us", "ms", "ns") else u[key])
        st = [(float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
              for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
              and v.replace(",", "").replace(".", "").isdigit()]
        tot = sum(v for v, _ in st) or 1.0
        k["top_stalls_pct"] = {h: round(100 * v / tot, 1) for v, h in sorted(st, reverse=True)[:6]}
        out.append(k)
    return out


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    res = {}
    for f in sorted(os.listdir(os.path.join(ROOT, "gpurun_out"))):
        if f.startswith("prof_") and f.endswith(".ncu-rep"):
            res[f[5:-8]] = summarize(os.path.join(ROOT, "gpurun_out", f))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:6000])
    # per-workload step-kernel figures read by bench.py (roofline.traffic)
    summ = {}
    for wl, ks in res.items():
        st = [k for k in ks if "step_tma_kernel" in k["kernel"]]
        if not st:
            continue
        summ[wl] = {"kernel": st[0]["kernel"],
                    "dram_bytes_per_launch": sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in st) / len(st),
                    "gpu_time_us_per_launch": sum(k["gpu__time_duration.sum"] for k in st) / len(st),
                    "source": (f"profiles/{tag}_ncu_full.json (ncu --set full, kernel replay, cache control all: "
                               "cold L2 per replay)") if "smsp__issue_active.avg.pct_of_peak_sustained_active" in st[0]
                    else (f"profiles/{tag}_ncu_full.json (ncu DRAM metrics only, application replay of the bench "
                          "command, launch after the warm-up: no memory save/restore of the working set)")}
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as fh:
        json.dump(summ, fh, indent=1)
