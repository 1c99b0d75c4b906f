"""Attribute ncu per-SASS-instruction execution counts and stall samples to
generated-source lines (the NVRTC source is not importable by ncu).
  python scripts/sass_lines.py REP.ncu-rep GEN.cubin GEN.cu [top]
The cubin is the same generated source compiled locally with nvcc -lineinfo
(scripts/check_codegen.py); instructions are matched by offset and opcode."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def main(rep, cubin, src, top=40):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    line = None
    loc = {}
    ops = {}
    for ln in dis.splitlines():
        m = re.search(r'//## File "(.*)", line (\d+)', ln)
        if m:
            line = int(m.group(2)) if m.group(1).endswith(".cu") and "gen" in m.group(1) else -int(m.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            off = int(m.group(1), 16)
            loc[off] = line
            ops[off] = m.group(2).split()[0] if not m.group(2).startswith("@") else m.group(2).split()[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    by_line = defaultdict(lambda: [0, 0])
    mism = 0
    tot_ex = tot_st = 0
    for r in rows[2:]:
        off = int(r[ia], 16) - base
        ex, st = int(r[iex] or 0), int(r[ist] or 0)
        tot_ex += ex
        tot_st += st
        op = r[isrc].strip().split()[0] if not r[isrc].strip().startswith("@") else r[isrc].strip().split()[1]
        if (ops.get(off) or "").split(".")[0] != op.split(".")[0]:
            mism += 1
        by_line[loc.get(off)][0] += ex
        by_line[loc.get(off)][1] += st
    text = open(src).read().splitlines()
    print("opcode mismatches: %d of %d" % (mism, len(rows) - 2))
    print("%6s %7s %7s  %s" % ("line", "inst%", "stall%", "source"))
    for l, (ex, st) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        s = text[l - 1].strip()[:90] if l and 0 < l <= len(text) else "(header line %s)" % l
        print("%6s %6.2f%% %6.2f%%  %s" % (l, 100.0 * ex / tot_ex, 100.0 * st / max(tot_st, 1), s))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
