"""Turn gpurun_out/{launches.csv, prof_final.ncu-rep} into the profiles/ summaries:
launch list shares, per-kernel DRAM traffic json, and the --set full details csv."""
import csv, collections, json, subprocess, sys

def launches(path, out):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[r[ii]]["k"] = r[ki]
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault(d["k"], [0.0, 0, 0.0, 0.0, 0.0])
        a[0] += d.get("gpu__time_duration.sum", 0) / 1e3
        a[1] += 1
        a[2] += d.get("smsp__inst_executed.sum", 0)
        a[3] += d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)
        a[4] += d.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0)
    # Engine kernels (shares of the engine's GPU time; the one-time map build
    # k_nnf_query / k_point_* and the bench's micro_peaks roofline kernels are
    # listed after them, without a share).
    def engine(k):
        return ("smcl::" in k or "cub::" in k) and "k_nnf_query" not in k
    tot = sum(a[0] for k, a in agg.items() if engine(k))
    with open(out, "w") as f:
        f.write("# engine kernels: share of engine GPU time, mean us per launch x launches, warp instructions per "
                "launch, achieved occupancy, active threads per instruction\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1][0]):
            if engine(k):
                f.write(f"{a[0] / tot * 100:5.1f}% {a[0] / a[1]:9.1f}us x{a[1]:3d} inst {a[2] / a[1] / 1e6:9.1f}M "
                        f"occ {a[3] / a[1]:5.1f}% thr/inst {a[4] / a[1]:5.1f} {k[:90]}\n")
        f.write("# other kernels in the same run (one-time map build, micro_peaks roofline kernels)\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1][0]):
            if not engine(k):
                f.write(f"     {a[0] / a[1]:9.1f}us x{a[1]:3d} inst {a[2] / a[1] / 1e6:9.1f}M {k[:90]}\n")

def traffic(rep, out, src):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    ki = h.index("Kernel Name")
    cols = {m: h.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                                    "sm__inst_issued.avg.per_cycle_active",
                                    "sm__inst_issued.avg.pct_of_peak_sustained_active")}
    units = rows[1]
    res = {}
    names = {"k_refresh_gather": "refresh_gather", "k_gicp_fast": "gicp_gn (K1)", "k_gicp_ll": "gicp_ll (K2)",
             "k_ll_count": "ll_count (K2a)", "k_svgd": "svgd (K8)", "k_smooth_round": "smooth round (K12)",
             "k_reorder": "reorder (K4)", "k_chunk_serial": "chunk serial sums (K11)"}
    def val(r, m):
        v = float(r[cols[m]].replace(",", ""))
        u = units[cols[m]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1)
        return v * scale
    for r in rows[2:]:
        for pat, nm in names.items():
            if pat in r[ki] and nm not in res:
                res[nm] = {"dram_read_bytes": val(r, "dram__bytes_read.sum"),
                           "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                           "ncu_duration_ms": val(r, "gpu__time_duration.sum"),
                           "ipc_issued": float(r[cols["sm__inst_issued.avg.per_cycle_active"]].replace(",", "")),
                           "issue_pct_of_peak": float(
                               r[cols["sm__inst_issued.avg.pct_of_peak_sustained_active"]].replace(",", "")),
                           "kernel": r[ki][:80]}
    json.dump({"source": src, "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))

if __name__ == "__main__":
    # summarize_profiles.py <launches.csv> <full.ncu-rep>[,<more.ncu-rep>] <round tag> <command>
    csv_path, reps, tag, cmd = sys.argv[1], sys.argv[2].split(","), sys.argv[3], sys.argv[4]
    launches(csv_path, f"profiles/{tag}_launch_summary.txt")
    merged = {}
    for rep in reps:
        traffic(rep, "/tmp/_traffic.json", cmd)
        merged.update(json.load(open("/tmp/_traffic.json"))["kernels"])
    json.dump({"source": f"ncu --set full --clock-control none, {cmd} ({tag})", "kernels": merged},
              open(f"profiles/{tag}_dram_traffic.json", "w"), indent=1)
