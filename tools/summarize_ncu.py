#!/usr/bin/env python3
"""Summarise a round's ncu evidence (gpurun_out/) into profiles/.

    python tools/summarize_ncu.py r1

Writes profiles/<tag>_launches.md (every launch of the profiled bench
command, grouped by kernel: count, total time, share of kernel time),
profiles/<tag>_kernels.md (full-set metrics of one iteration's worth of each
hot kernel) and profiles/ncu_traffic.json (average DRAM bytes per launch per
bench kernel kind, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KIND = [  # bench.py kernel kind <- short ncu name prefixes
    ("K1_grad_limit", "k_grad_limit<"),
    ("K1_grad_limit", "k_grad_limit_brick<"),
    ("K2_face_pred", "k_face_flux<Euler3D, 1"),
    ("K2_face_corr", "k_face_flux<Euler3D, 0"),
    ("K3_update_pred", "k_gather_update<Euler3D, 1, 0"),
    ("K3_update_corr", "k_gather_update<Euler3D, 0"),
]

UNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kind_of(name):
    n = short(name)
    for k, frag in KIND:
        if n.startswith(frag):
            return k
    return None


def short(name):
    return name.replace("void ", "").replace("tafv::", "").split("(")[0]


def launch_rows(tag):
    """{launch id: {"name", metric: value in base units}} from a launch list
    (one or several metrics per launch; ncu's preamble lines skipped)."""
    lines = open(os.path.join(OUT, f"launches_{tag}.csv")).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = per.setdefault(r[ix["ID"]], {"name": short(r[ix["Kernel Name"]])})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1.0)
    return per


def launches(tag, what):
    per = launch_rows(tag)
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    dram = any(v[2] for v in agg.values())
    lines = [f"# {tag}: ncu launch list of `{what}`",
             "", "`ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --clock-control none`",
             "(cold-cache, serialised launches: compare SHARES with bench.py's event-timed breakdown, not absolutes).", "",
             "| kernel | launches | total us | share of kernel time | avg us |" + (" DRAM GB | DRAM TB/s |" if dram else ""),
             "|---|---|---|---|---|" + ("---|---|" if dram else "")]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        row = f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / tot * 100:.1f} % | {v[1] / v[0]:.1f} |"
        if dram:
            row += f" {v[2] / 1e9:.2f} | {v[2] / max(v[1], 1e-9) / 1e6:.2f} |"
        lines.append(row)
    lines.append(f"| **all** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100 % | |" + (" | |" if dram else ""))
    return "\n".join(lines) + "\n"


def launch_traffic(tag):
    """Mean DRAM bytes per launch of each bench kernel kind over the launch
    list (every launch of the profiled iteration), when it carries DRAM bytes."""
    per = launch_rows(tag)
    tr = {}
    for d in per.values():
        if "dram__bytes_read.sum" not in d:
            return {}
        kind = kind_of(d["name"])
        if kind:
            tr.setdefault(kind, []).append(d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0))
    return {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v),
                "source": f"profiles/{tag}_launches.md (ncu launch list, cold cache, mean over every launch of the "
                          "profiled iteration)"} for k, v in tr.items()}


METRICS = [  # (metric, column, scale from base units: ns / bytes)
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1e-6),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak", 1),
    ("launch__registers_per_thread", "regs/thread", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("launch__grid_size", "grid", 1),
]


def raw_rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def val(r, hdr, units, m):
    """Metric value in base units (ns, bytes) using the CSV unit row."""
    if m not in hdr:
        return None
    i = hdr.index(m)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return None
    return v * UNIT.get(units[i], 1.0)


def full(tag):
    lines = [f"# {tag}: ncu --set full captures (gpurun_out/full_{tag}*.ncu-rep)", "",
             "`ncu --set full --clock-control none --import-source on -k regex:<kernels> [-c N]` on the",
             "profiled command of the launch list (cache flushed between replays: cold-cache numbers).", ""]
    traffic = {}
    import glob
    for rep in sorted(glob.glob(os.path.join(OUT, f"full_{tag}*.ncu-rep"))):
        k = os.path.basename(rep)[len(f"full_{tag}"):-len(".ncu-rep")].strip("_") or tag
        hdr, units, rows = raw_rows(rep)
        lines += [f"## `{k}`", "", "| launch | kernel | " + " | ".join(m[1] for m in METRICS) + " | top stalls (cycles/issue) |",
                  "|---" * (len(METRICS) + 3) + "|"]
        for i, r in enumerate(rows):
            name = r[hdr.index("Kernel Name")]
            vals = []
            for m, _, sc in METRICS:
                v = val(r, hdr, units, m)
                vals.append("-" if v is None else f"{v * sc:.1f}")
            st = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                          float(r[j] or 0)) for j, h in enumerate(hdr)
                         if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")),
                        key=lambda x: -x[1])[:3]
            lines.append(f"| {i} | `{short(name)}` | " + " | ".join(vals) + " | " +
                         ", ".join(f"{a} {b:.1f}" for a, b in st) + " |")
            kind = kind_of(name)
            if kind:
                b = val(r, hdr, units, "dram__bytes_read.sum") + val(r, hdr, units, "dram__bytes_write.sum")
                traffic.setdefault(kind, []).append(b)
        lines.append("")
    tj = {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v),
              "source": f"profiles/{tag}_kernels.md (ncu --set full, cold cache, mean over the captured launches)"}
          for k, v in traffic.items()}
    return "\n".join(lines) + "\n", tj


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    what = sys.argv[2] if len(sys.argv) > 2 else "python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1"
    os.makedirs(PROF, exist_ok=True)
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write(launches(tag, what))
    md, tj = full(tag)
    open(os.path.join(PROF, f"{tag}_kernels.md"), "w").write(md)
    tj.update(launch_traffic(tag))  # every launch of the iteration beats a sample of launches
    json.dump(tj, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    main()
