"""Write profiles/<tag>_ncu_evidence.md (run here, no GPU): for each kernel choice of SURVEY 8(d),
the ncu counters of the committed --set full captures (profiles/<tag>_ncu_full.json) next to the
SASS facts of the built library (cuobjdump): bulk copies, 128-bit accesses, shuffles, tensor-core
instructions."""
import collections, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
LIB = os.path.join(ROOT, "paper_2309_12381_b200", "lib", "libmpo.so")
BYTES = {"resnet50_sgd": (25557032, 10, 8), "gpt2_adamw": (124439808, 14, 12), "vit_l16_adam_clip": (304326632, 14, 12)}

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = collections.defaultdict(list), None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and cur:
        funcs[cur].append(m.group(1))


def count(pred, name_re):
    return {f: sum(1 for op in ops if pred(op)) for f, ops in funcs.items() if re.search(name_re, f)}


def agg(d):
    return (min(d.values()), max(d.values())) if d else (0, 0)


tensor = lambda op: op.startswith(("HMMA", "IMMA", "UTCMMA", "UTCHMMA", "UTCQMMA", "QMMA", "OMMA", "HGMMA"))
rows = []
for fam, rx in (("step_tma_kernel", r"step_tma_kernel"), ("sumsq_kernel", r"sumsq_kernel"),
                ("sumsq_tma_kernel", r"sumsq_tma_kernel"), ("split_kernel", r"split_kernel"),
                ("reconstruct_kernel", r"reconstruct_kernel"), ("p2p_step_kernel", r"p2p_step_kernel"),
                ("nvls_step_kernel", r"nvls_step_kernel")):
    n = len([f for f in funcs if re.search(rx, f)])
    if not n:
        continue
    rows.append((fam, n, agg(count(lambda op: op.startswith("UBLKCP"), rx)),
                 agg(count(lambda op: op.startswith(("LDG", "STG")) and op.endswith(".128"), rx)),
                 agg(count(lambda op: op.startswith("SHFL"), rx)), agg(count(tensor, rx)),
                 agg(count(lambda op: op.startswith("LDGMC") or op.endswith(".STRONG.SYS"), rx))))

full = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.json")))
out = [f"# {tag}: ncu + SASS evidence per kernel choice (SURVEY.md 8(d))", "",
       f"Counters: `profiles/{tag}_ncu_full.json` (ncu --set full, cold L2 per replay, one B200).",
       f"SASS: `cuobjdump -sass {os.path.relpath(LIB, ROOT)}` (all instantiations; min-max per family).", "",
       "## ncu, step kernel and clip pre-pass", "",
       "| workload | kernel | us | DRAM R / W (MB) | algorithmic R / W (MB) | DRAM % of peak | issue active % | warps active % | regs | store sectors/request | tensor pipe % | top stalls |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for wl, ks in full.items():
    for k in ks:
        name = k["kernel"].split("(")[0].replace("void ", "")
        if "final" in name:
            continue
        P, rb, wb = BYTES.get(wl, (0, 0, 0))
        if "sumsq" in name:
            rb, wb = 2, 0
        st_s = k.get("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", 0)
        st_r = k.get("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", 1) or 1
        stalls = ", ".join(f"{a} {b}" for a, b in list(k.get("top_stalls_pct", {}).items())[:3])
        out.append(f"| {wl} | `{name}` | {k['gpu__time_duration.sum']:.1f} | "
                   f"{k['dram__bytes_read.sum'] / 1e6:.0f} / {k['dram__bytes_write.sum'] / 1e6:.0f} | "
                   f"{P * rb / 1e6:.0f} / {P * wb / 1e6:.0f} | "
                   f"{k.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                   f"{k.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                   f"{k.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                   f"{k.get('launch__registers_per_thread', 0):.0f} | {st_s / st_r:.1f} | "
                   f"{k.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | {stalls} |")
out += ["", "Reading: DRAM bytes = the algorithmic bytes (no over-fetch; writes slightly below because the",
        "last dirty lines are still in L2 when the replay ends); the tensor pipe is idle (no contraction);",
        "issue stays well below peak (not ALU-bound). Store sectors/request: 16 for the 16-bit streams,",
        "32 half sectors for each of the two 128-bit fp32 stores of a unit (256-bit stores were measured",
        "and rejected, profiles/r01_ab13_st256.log). ncu's DRAM '% of peak' is against the nominal",
        "peak; the bench reports against the measured copy peak (MEASURED_PEAKS.json).", "",
        "## SASS facts (min-max over the family's instantiations)", "",
        "| kernel family | instantiations | UBLKCP (TMA bulk copy) | 128-bit LDG/STG | SHFL | tensor-core instr | multimem (LDGMC + STG...STRONG.SYS) |",
        "|---|---|---|---|---|---|---|"]
for fam, n, ub, v128, sh, tc, mc in rows:
    f = lambda t: f"{t[0]}" if t[0] == t[1] else f"{t[0]}-{t[1]}"
    out.append(f"| `{fam}` | {n} | {f(ub)} | {f(v128)} | {f(sh)} | {f(tc)} | {f(mc)} |")
out += ["", "Shuffles appear only in the global-norm pre-pass (`sumsq_*`); no kernel issues a tensor-core",
        "instruction; the default step kernel moves every input stream with bulk copies (UBLKCP) and",
        "stores with 128-bit STG; the multicast kernel reduces with LDGMC (multimem.ld_reduce) and",
        "stores through the multicast address (multimem.st -> STG.E.128.STRONG.SYS); the P2P kernel's",
        "peer loads/stores are ordinary 128-bit LDG/STG on peer addresses."]
path = os.path.join(ROOT, "profiles", f"{tag}_ncu_evidence.md")
open(path, "w").write("\n".join(out) + "\n")
print(path)
