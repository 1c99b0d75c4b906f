"""Summarise ncu captures for profiles/: key raw metrics, opcode mix weighted by
executed instructions, lane efficiency, instructions per SSA event.

  python scripts/ncu_summary.py OUT.md rep1.ncu-rep[:events] [rep2.ncu-rep[:events] ...]
  (events = SSA events processed by the captured launch, for per-event figures)
  python scripts/ncu_summary.py OUT.md --launches launches.csv
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of peak)"),
    ("smsp__warps_active.avg.per_cycle_active", "warps active per SMSP"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "SM issue active (% of peak)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe (%)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (%)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe (%)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (%)"),
    ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (% elapsed)"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep, events):
    lines = []
    raw = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = raw[0], raw[1]
    for r in raw[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append("### %s — `%s`\n" % (rep.split("/")[-1], name))
        lines.append("| metric | value |\n|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append("| %s (`%s`) | %s %s |" % (label, m, r[i], units[i]))
        lines.append("")
    src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        iS, iE, iT = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
        iW = h.index("Warp Stall Sampling (All Samples)")
        tot = tott = totw = 0
        op, opw = collections.Counter(), collections.Counter()
        for r in src[2:]:
            try:
                e, t, w = int(r[iE]), int(r[iT]), int(r[iW])
            except (ValueError, IndexError):
                continue
            s = r[iS].split()
            o = (s[1] if s and s[0].startswith("@") and len(s) > 1 else (s[0] if s else "?")).split(".")[0]
            op[o] += e
            opw[o] += w
            tot += e
            tott += t
            totw += w
        lines.append("lane efficiency (thread inst / 32 warp inst): **%.3f**" % (tott / max(tot, 1) / 32))
        if events:
            lines.append("; SSA events in this launch: %d; **warp-instructions per event: %.1f**, "
                         "thread-instructions per event: %.1f" % (events, tot / events, tott / events))
        lines.append("\n| opcode | % of executed warp inst | % of stall samples |\n|---|---|---|")
        for o, e in op.most_common(16):
            lines.append("| %s | %.1f | %.1f |" % (o, 100 * e / tot, 100 * opw[o] / max(totw, 1)))
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > v:
            tot.setdefault(r[k], []).append(float(r[v]))
    allt = sum(sum(x) for x in tot.values())
    out = ["| kernel | launches | total ns | share |", "|---|---|---|---|"]
    for n, x in tot.items():
        out.append("| %s | %d | %.0f | %.1f %% |" % (n[:60], len(x), sum(x), 100 * sum(x) / allt))
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    out = sys.argv[1]
    parts = []
    if sys.argv[2] == "--launches":
        parts.append(launches(sys.argv[3]))
    else:
        for a in sys.argv[2:]:
            rep, _, ev = a.partition(":")
            parts.append(summarize(rep, int(ev) if ev else 0))
    with open(out, "w") as fh:
        fh.write("\n".join(parts))
    print(open(out).read())
