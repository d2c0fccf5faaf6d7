"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

  python profiles/summarize.py ROUND gpurun_out/prof_k1.ncu-rep gpurun_out/launches.csv
  python profiles/summarize.py --late ROUND gpurun_out/prof_late.ncu-rep paper_2602_22421_b200/libspfom.so

writes profiles/<ROUND>_k1_full.txt (key metrics, stall reasons, instruction
mix), profiles/<ROUND>_launches.csv (the per-launch list) and updates
profiles/ncu_summary.json (DRAM bytes per K1 launch, read by bench.py's
roofline.traffic; key k_primal for huge, k_primal@<WORKLOAD> for the other
configs -- set WORKLOAD=medium|multi when summarising their captures).
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_red.sum",
        "smsp__inst_executed_op_global_red.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        res.append(d)
    return res


def sass_profile(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[1], rows[2:]
    iI, iS, iSrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot_s = sum(float(r[iS] or 0) for r in data) or 1.0
    stalls = {c: sum(float(r[h.index(c)] or 0) for r in data) / tot_s * 100 for c in stall_cols}
    tot_i = sum(float(r[iI] or 0) for r in data) or 1.0
    ops = collections.Counter()
    for r in data:
        s = re.sub(r"^@!?U?P\w+\s+", "", r[iSrc].strip())
        ops[s.split(" ")[0] if s else "?"] += float(r[iI] or 0)
    mix = {k: v / tot_i * 100 for k, v in ops.most_common(20)}
    sass_tags = sorted({op for op in ops if re.match(r"(UTC|UBLK|UTMA|LDTM|STTM|HMMA|REDG|RED|ATOM)", op)})
    return stalls, mix, sass_tags


ITER_KERNELS = ("k_primal", "k_fold", "k_dual", "k_tick", "k_average")   # launched every iteration


def write_launch_summary(rnd, path):
    """Per-kernel launch counts and average gpu__time_duration from an ncu
    --metrics gpu__time_duration.sum launch list; shares of one iteration."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4]
        agg.setdefault(name, []).append(float(r[14]) / 1e3)      # us
    it_total = sum(sum(v) / len(v) for k, v in agg.items()
                   if any(x in k for x in ITER_KERNELS))
    lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none launch list ({os.path.basename(path)}),",
             "cold-cache and serialised: compare shares, not absolutes.  Per-iteration kernels: " +
             ", ".join(ITER_KERNELS) + "; k_usage / k_resid_* run once for the residuals call outside the timed loop.",
             ""]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        avg = sum(v) / len(v)
        per_iter = any(x in k for x in ITER_KERNELS)
        share = f"{avg / it_total * 100:5.1f}% of iteration" if per_iter and it_total else "(not in the iteration)"
        lines.append(f"  {len(v):4d} launches  avg {avg:9.1f} us   {share}  {k}")
    open(os.path.join(HERE, f"{rnd}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def write_late(rnd, rep, so):
    """Steady-state capture (exp/prof_late.sh, iteration ~1500): key metrics,
    stall reasons and the source lines that take the most stall samples, from
    the SASS source page mapped to CUDA lines through `nvdisasm -g` of the
    library that ran (`so`)."""
    import tempfile
    mets = raw_metrics(rep)
    stalls, mix, _ = sass_profile(rep)
    kname = mets[0]["kernel"]
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    mangled = None
    for ln in dis.splitlines():
        if ln.startswith("//----") and "k_primal_stream" in ln and "Lb0ELi13E" in ln:
            mangled = ln.split(".text.")[1].split()[0]
            break
    off2loc, cur, inside = {}, None, False
    for ln in dis.splitlines():
        if ln.startswith("//----"):
            inside = mangled is not None and mangled in ln
            continue
        if not inside:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m:
            off2loc[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[1], rows[2:]
    iI, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    base = None
    for r in data:
        if not r or not r[0].startswith("0x"):
            continue
        a = int(r[0], 16)
        base = a if base is None else base
        loc = off2loc.get(a - base)
        agg[loc][0] += float(r[iI] or 0)
        agg[loc][1] += float(r[iS] or 0)
    ti = sum(v[0] for v in agg.values()) or 1.0
    ts = sum(v[1] for v in agg.values()) or 1.0
    src = {}
    lines = [f"ncu --set full of one K1 launch in the steady state ({os.path.basename(rep)}), round {rnd}", "",
             f"kernel: {kname}"]
    for k in KEYS:
        if k in mets[0]:
            lines.append(f"  {k:62s} {mets[0][k][0]} {mets[0][k][1]}")
    lines += ["", "stall reasons (% of samples): " + ", ".join(f"{k} {v:.1f}" for k, v in
                                                            sorted(stalls.items(), key=lambda x: -x[1])[:10]),
              "", "source lines by stall samples (% samples, % instructions):"]
    for loc, (n, smp) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        text = ""
        if loc:
            if loc[0] not in src:
                pth = os.path.join(os.path.dirname(HERE), "paper_2602_22421_b200", "csrc", loc[0])
                src[loc[0]] = open(pth).read().splitlines() if os.path.exists(pth) else []
            if loc[1] - 1 < len(src[loc[0]]):
                text = src[loc[0]][loc[1] - 1].strip()[:80]
        lines.append(f"  {smp / ts * 100:5.1f}% {n / ti * 100:5.1f}%  {loc[0] if loc else '?'}:{loc[1] if loc else ''}  {text}")
    open(os.path.join(HERE, f"{rnd}_k1_late.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def main():
    if sys.argv[1] == "--late":
        write_late(sys.argv[2], sys.argv[3], sys.argv[4])
        return
    rnd, rep = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    mets = raw_metrics(rep)
    stalls, mix, tags = sass_profile(rep)
    lines = [f"ncu --set full capture of K1 ({os.path.basename(rep)}), round {rnd}", ""]
    for m in mets:
        lines.append(f"kernel: {m['kernel']}")
        for k in KEYS:
            if k in m:
                lines.append(f"  {k:62s} {m[k][0]} {m[k][1]}")
    lines.append("")
    lines.append("stall reasons (% of samples): " + ", ".join(f"{k} {v:.1f}" for k, v in
                                                            sorted(stalls.items(), key=lambda x: -x[1])[:10]))
    lines.append("instruction mix (% of executed): " + ", ".join(f"{k} {v:.1f}" for k, v in mix.items()))
    lines.append("notable SASS ops present: " + ", ".join(tags))
    open(os.path.join(HERE, f"{rnd}_k1_full.txt"), "w").write("\n".join(lines) + "\n")
    m = mets[0]
    rd = float(m["dram__bytes_read.sum"][0]) * UNIT[m["dram__bytes_read.sum"][1]]
    wr = float(m["dram__bytes_write.sum"][0]) * UNIT[m["dram__bytes_write.sum"][1]]
    summ_path = os.path.join(HERE, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    wl = os.environ.get("WORKLOAD", "huge")
    summ["k_primal" if wl == "huge" else f"k_primal@{wl}"] = {"round": rnd, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                        "duration": m["gpu__time_duration.sum"], "source": os.path.basename(rep),
                        "workload": wl,
                        # COVERS_K1=0: the capture is one of several concurrent bin launches
                        # (medium), so its bytes are not the K1 step's traffic
                        "covers_k1": os.environ.get("COVERS_K1", "1") == "1"}
    json.dump(summ, open(summ_path, "w"), indent=1)
    if launches:
        shutil.copy(launches, os.path.join(HERE, f"{rnd}_launches.csv"))
        write_launch_summary(rnd, launches)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
