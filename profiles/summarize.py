#!/usr/bin/env python3
"""Summaries of the ncu captures kept under profiles/ (run here, not on the GPU box).

    python profiles/summarize.py launches <launches.csv> <out.md>
        per-kernel time per step from an `ncu --metrics gpu__time_duration.sum
        --clock-control none --csv` launch list of `python bench.py`; the bench
        runs 8 distinct balanced mini-batches (slots) per epoch, so the summary
        averages the first 8 complete post-warm-up steps.
    python profiles/summarize.py full <capture.ncu-rep> <out.md> [N P]
        per-launch duration, DRAM traffic, throughput, occupancy, issue
        utilisation and pipe activity of every kernel in an `ncu --set full`
        capture; with the step's atoms N and edges P, the algorithmic bytes of
        the edge kernels (bench.kernel_bytes) next to the measured DRAM bytes.
    python profiles/summarize.py traffic <capture.ncu-rep> <out.json> N P section
        DRAM bytes per launch of each edge / GEMM kernel of the capture's last step
        next to the algorithmic and compulsory bytes, merged into out.json under
        `section` (bench.py reads roofline.traffic from it).
"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _rows(text):
    rows = list(csv.reader(io.StringIO(text)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def launches(path, out):
    data = _rows(open(path).read())
    steps, cur = [], []
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        if name.startswith("k_prep") and cur:
            steps.append(cur)
            cur = []
        cur.append((name, float(d["Metric Value"]) / 1e3))
    steps.append(cur)
    full = [s for s in steps if s and s[0][0].startswith("k_prep")]
    sel = full[:8]
    agg = collections.OrderedDict()
    for s in sel:
        for name, t in s:
            a = agg.setdefault(name, [0.0, 0])
            a[0] += t
            a[1] += 1
    tot = sum(v[0] for v in agg.values())
    lines = [f"# Launch list summary ({os.path.basename(path)})", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold caches):",
             f"{len(sel)} complete steps averaged (the 8 balanced mini-batches of the epoch), "
             f"{len(sel[0]) if sel else 0} launches per step.", "",
             "| kernel | us / step | launches / step | share |", "|---|---:|---:|---:|"]
    for name, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {name} | {t / len(sel):.1f} | {n / len(sel):.0f} | {100 * t / tot:.1f}% |")
    lines += ["", f"Sum of kernel durations per step: {tot / len(sel):.1f} us "
                  f"(per-step totals: {', '.join(f'{sum(t for _, t in s):.0f}' for s in sel)} us)."]
    open(out, "w").write("\n".join(lines) + "\n")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size"]


def full(path, out, N=None, P=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    kb = None
    if N is not None:
        import bench
        kb = bench.kernel_bytes
    short = {"k_edge_bwd": "bwd_edge", "k_edge_message": "message", "k_edge_head": "head_bwd",
             "k_edge_force": "force", "k_node_gemm": "update", "k_dwu": "dwu"}
    lines = [f"# ncu --set full summary ({os.path.basename(path)})", ""]
    if N is not None:
        lines.append(f"Step captured: N = {N} atoms, P = {P} directed edges.")
        lines.append("")
    lines += ["| kernel | us | DRAM rd MB | DRAM wr MB | algorithmic MB | DRAM % peak | SM % | issue % | "
              "FMA pipe % | tensor pipe % | L2 hit % | warps active % | regs |",
              "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]

    def g(r, m, scale=1.0):
        if m not in idx:
            return float("nan")
        try:
            v = float(r[idx[m]].replace(",", ""))
        except ValueError:
            return float("nan")
        u = units[idx[m]]
        if m.startswith("dram__bytes") or m == "lts__t_bytes.sum":
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
        return v * scale

    for r in data:
        name = r[kn].split("(")[0].replace("void ", "").replace("lamm_b200::", "")
        base = name.split("<")[0]
        alg = ""
        if kb and base in short and kb(short[base], N, P) is not None:
            alg = f"{kb(short[base], N, P) / 1e6:.1f}"
        lines.append(
            f"| {name} | {g(r, 'gpu__time_duration.sum'):.1f} | {g(r, 'dram__bytes_read.sum') / 1e6:.2f} | "
            f"{g(r, 'dram__bytes_write.sum') / 1e6:.2f} | {alg} | "
            f"{g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'lts__t_sector_hit_rate.pct'):.1f} | "
            f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'launch__registers_per_thread'):.0f} |")
    lines += ["", "ncu flushes caches before every replayed kernel (--cache-control all), so DRAM bytes are the",
              "compulsory traffic of one launch; writes still sitting in L2 at kernel end are not counted."]
    open(out, "w").write("\n".join(lines) + "\n")


SHORT = {"k_edge_message": "message", "k_message_update": "message", "k_edge_force": "force", "k_edge_head": "head_bwd", "k_edge_bwd": "bwd_edge",
         "k_node_gemm": "update", "k_bwd_gemm": "bwd_gemm"}


def _merge(out, section, path, N, P, acc):
    import json
    import bench
    doc = json.load(open(out)) if os.path.exists(out) else {}
    res = {"source": f"ncu --set full --clock-control none (cache flush before each replayed kernel), "
                     f"{os.path.basename(path)}; the last step's launches", "N": N, "P": P, "kernels": {}}
    for name, (n, t, d) in acc.items():
        alg, uniq = bench.kernel_bytes(name, N, P), bench.kernel_bytes_unique(name, N, P)
        res["kernels"][name] = {"launches": n, "dram_bytes": t / n, "us_cold": d / n, "algorithmic_bytes": alg,
                                "compulsory_bytes": uniq, "dram_over_algorithmic": t / n / alg,
                                "dram_over_compulsory": t / n / uniq}
    doc[section] = res
    json.dump(doc, open(out, "w"), indent=1)


def traffic_md(path, out, N, P, section):
    rows = [ln.split("|")[1:-1] for ln in open(path) if ln.startswith("| k_")]
    start = max(i for i, r in enumerate(rows) if r[0].strip() == "k_prep")
    acc = collections.OrderedDict()
    for r in rows[start:]:
        name = SHORT.get(r[0].strip().split("<")[0])
        if name is None:
            continue
        us, rd, wr = float(r[1]), float(r[2]) * 1e6, float(r[3]) * 1e6
        n, t, d = acc.get(name, (0, 0.0, 0.0))
        acc[name] = (n + 1, t + rd + wr, d + us)
    _merge(out, section, path, N, P, acc)


def traffic(path, out, N, P, section):
    """Per edge/GEMM kernel of the LAST step in the capture: DRAM bytes per launch
    next to SURVEY §8(d)'s algorithmic (gather-inclusive) bytes and the compulsory
    bytes (bench.kernel_bytes / kernel_bytes_unique); merged into `out` under
    `section` (bench.py reads roofline.traffic from it)."""
    import json
    import bench
    if path.endswith(".md"):  # a `full` summary table (the capture itself stayed on the GPU box)
        return traffic_md(path, out, N, P, section)
    if path.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` output
        txt = open(path).read()
    else:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kn, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    du = hdr.index("gpu__time_duration.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
             "ns": 1e-3, "us": 1.0, "ms": 1e3}
    short = SHORT
    # the last step: from the last k_prep on
    start = max(i for i, r in enumerate(data) if "k_prep" in r[kn])
    acc = collections.OrderedDict()
    for r in data[start:]:
        name = short.get(r[kn].split("<")[0].split("(")[0].strip().split(" ")[-1])
        if name is None:
            continue
        b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
        us = float(r[du].replace(",", "")) * scale[units[du]]
        n, t, d = acc.get(name, (0, 0.0, 0.0))
        acc[name] = (n + 1, t + b, d + us)
    _merge(out, section, path, N, P, acc)


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        n = int(sys.argv[4]) if len(sys.argv) > 4 else None
        p = int(sys.argv[5]) if len(sys.argv) > 5 else None
        full(sys.argv[2], sys.argv[3], n, p)
