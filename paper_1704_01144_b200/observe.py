"""Observability: per-iteration records as CSV and the
paper's level-occupancy tables (cell share / cost share per level,
PAPER.md Tables 1-3; cost model C(tau) = 2^(theta-tau)|Omega(tau)|,
levels.cpp:68-79). NVTX ranges ("tafv.plan", "tafv.sweep", "tafv.phase.*")
are emitted by the library itself."""
from __future__ import annotations

import csv


def level_table(record):
    """[(tau, cells, cell share %, cost share %)] for one IterationRecord."""
    th = record["theta"]
    cells = record["level_cells"]
    cost = [n << (th - l) for l, n in enumerate(cells)]
    nc, tc = sum(cells), sum(cost)
    return [(l, n, 100.0 * n / nc if nc else 0.0, 100.0 * c / tc if tc else 0.0)
            for l, (n, c) in enumerate(zip(cells, cost))]


def format_level_table(record):
    rows = ["| tau | cells | cells % | cost % |", "|---|---|---|---|"]
    for l, n, cs, ks in level_table(record):
        rows.append(f"| {l} | {n} | {cs:.3f} | {ks:.3f} |")
    rows.append(f"cost ratio (2^theta N / sum C) = {record['cost_ratio']:.4f}")
    return "\n".join(rows)


def records_to_csv(records, path, kernel_times=None):
    """One row per IterationRecord (reference.hpp:20-29) + level/cost shares;
    optional per-kernel device times (Solver.kernel_times()) as extra columns
    of the last row's summary."""
    maxl = max((r["theta"] for r in records), default=0) + 1
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        hdr = ["iteration", "t_start", "dt", "theta", "advance", "cost_ratio"]
        hdr += [f"total_extensive_{k}" for k in range(len(records[0]["total_extensive"]))] if records else []
        hdr += [f"cells_tau{l}" for l in range(maxl)] + [f"cost_share_tau{l}" for l in range(maxl)]
        w.writerow(hdr)
        for r in records:
            tab = level_table(r)
            cells = [n for _, n, _, _ in tab] + [0] * (maxl - len(tab))
            shares = [round(ks, 6) for _, _, _, ks in tab] + [0.0] * (maxl - len(tab))
            w.writerow([r["iteration"], repr(r["t_start"]), repr(r["dt"]), r["theta"], repr(r["advance"]),
                        repr(r["cost_ratio"])] + [repr(x) for x in r["total_extensive"]] + cells + shares)
        if kernel_times:
            w.writerow([])
            w.writerow(["kernel", "ms", "launches"])
            for k, v in kernel_times.items():
                w.writerow([k, repr(v["ms"]), v["launches"]])
