"""Condense ncu reports into profiles/: per-kernel DRAM traffic + limiter metrics (JSON) and a
launch-list summary (text). Usage:
  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv --out profiles/r01
"""
import argparse, csv, collections, io, json, os, re, subprocess

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_tag_requests_pct": "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
    "l1_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_shared_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm_clock_mhz": "smsp__cycles_elapsed.avg.per_second",
    # the L2 <-> SM path the x gathers use
    "l1tex2xbar_req_cycles_active_pct": "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex2xbar_req_cycles_active_max_pct": "l1tex__m_l1tex2xbar_req_cycles_active.max.pct_of_peak_sustained_elapsed",
    "xbar2l1tex_read_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "xbar2l1tex_read_bytes_pct": "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
    "xbar2l1tex_read_sectors_pct": "l1tex__m_xbar2l1tex_read_sectors.avg.pct_of_peak_sustained_elapsed",
    "xbar2l1tex_tma_bytes": "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "xbar2l1tex_ldg_sectors": "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
UNITS = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "second": 1e6, "hz": 1e-6, "Khz": 1e-3, "Mhz": 1, "Ghz": 1e3}


def short(name):
    m = re.match(r"(?:void\s+)?(?:mcr::)?(\w+)(?:<\(?(?:int\)?)?(\d+)>)?", name)
    if not m:
        return name[:40]
    epi = {"0": "EPI_Y", "1": "EPI_RESID", "2": "EPI_JACOBI", "3": "EPI_S0", "4": "EPI_V", "5": "EPI_T"}
    ph = {"0": "PH_A", "1": "PH_C", "2": "PH_E"}
    k, t = m.group(1), m.group(2)
    if t is None:
        return k
    if k in ("k_spmv", "k_dense"):
        return f"{k}<{epi.get(t, t)}>"
    if k == "k_phase":
        return f"{k}<{ph.get(t, t)}>"
    return f"{k}<{t}>"


def rep_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    per = collections.defaultdict(list)
    for r in rows[2:]:
        d = {}
        for k, col in KEYS.items():
            if col in h:
                i = h.index(col)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * UNITS.get(u[i], 1.0) if k in ("duration_us", "dram_read_bytes", "dram_write_bytes", "sm_clock_mhz", "xbar2l1tex_read_bytes", "xbar2l1tex_tma_bytes") else v
        per[short(r[h.index("Kernel Name")])].append(d)
    kern = {}
    for k, lst in per.items():
        avg = {m: sum(x.get(m, 0) for x in lst) / len(lst) for m in KEYS}
        avg["dram_bytes_per_launch"] = avg["dram_read_bytes"] + avg["dram_write_bytes"]
        avg["captured_launches"] = len(lst)
        kern[k] = avg
    return kern


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[short(r[ki])].append(float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{'kernel':28s} {'launches':>8s} {'mean_us':>9s} {'total_us':>11s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:28s} {len(v):8d} {sum(v)/len(v):9.2f} {sum(v):11.1f} {sum(v)/tot:6.3f}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    kern = {}
    for r in a.rep:
        kern.update(rep_summary(r))
    if kern:
        with open(a.out + "_ncu.json", "w") as fh:
            json.dump({"note": a.note, "kernels": kern}, fh, indent=1, sort_keys=True)
    for i, l in enumerate(a.launches):
        with open(a.out + f"_launches{'' if i == 0 else i}.txt", "w") as fh:
            fh.write(f"# {a.note}\n# source: {os.path.basename(l)} (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)\n")
            fh.write(launches_summary(l))
