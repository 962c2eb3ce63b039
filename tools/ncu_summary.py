#!/usr/bin/env python3
"""Summarise ncu reports (.ncu-rep) and a launch list into a markdown file.

    python tools/ncu_summary.py gpurun_out profiles/r01_ncu_summary.md
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "TC smem operand wavefronts %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 tensor datapath active % (of active cycles)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        d["_units"] = dict(zip(head, units))
        recs.append(d)
    return recs


def stalls(d: dict) -> str:
    items = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                items.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    items.sort(reverse=True)
    tot = sum(v for v, _ in items) or 1.0
    return ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in items[:4])


def main() -> int:
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    lines = ["# ncu summaries", "", f"source: `{src}` (captured with `--set full --clock-control none`; "
             "times under ncu are serialised/replayed, never bench numbers)", ""]
    for rep in sorted(src.glob("*.ncu-rep")):
        for d in raw(rep):
            lines.append(f"## {rep.stem}: `{d.get('Kernel Name', '?')[:100]}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for k, label in KEYS:
                for cand in (k, "TPC.TriageCompute." + k):
                    if cand in d:
                        lines.append(f"| {label} (`{k}`) | {d[cand]} {d['_units'].get(cand, '')} |")
                        break
            lines.append(f"| top stall reasons | {stalls(d)} |")
            lines.append("")
    launches = src / "launches.csv"
    if launches.exists():
        text = launches.read_text().splitlines()
        start = next((i for i, l in enumerate(text) if l.startswith('"ID"')), None)
        if start is not None:
            rows = list(csv.DictReader(text[start:]))
            agg: dict[str, list[float]] = {}
            for r in rows:
                name = r.get("Kernel Name", "?")
                try:
                    agg.setdefault(name, []).append(float(r.get("Metric Value", "0")))
                except ValueError:
                    pass
            total = sum(sum(v) for v in agg.values()) or 1.0
            lines += ["## launch list (bench.py under ncu, per-kernel share of device time)", "",
                      "| kernel | launches | total | share |", "|---|---|---|---|"]
            for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:25]:
                lines.append(f"| `{name[:90]}` | {len(v)} | {sum(v):.0f} | {100 * sum(v) / total:.1f}% |")
            lines.append("")
            profiled = {d.get("Kernel Name", "?") for rep in sorted(src.glob("*.ncu-rep")) for d in raw(rep)}
            lines += ["Share of the step for the kernels captured above (cold-cache, serialised):", ""]
            for name in sorted(profiled):
                v = agg.get(name, [])
                lines.append(f"* `{name[:90]}`: {len(v)} launches, {sum(v):.0f} ns, {100 * sum(v) / total:.2f}% "
                             f"of the step, mean {sum(v) / max(1, len(v)):.0f} ns/launch")
            lines.append("")
    dst.write_text("\n".join(lines) + "\n")
    print(f"wrote {dst}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
