"""Per generated-source-line shared-memory wavefronts (total / excessive from bank conflicts)
of an ncu capture, matched to the dumped cubin's line table (as sass_lines.py).
  python scripts/smem_lines.py REP.ncu-rep GEN.cubin GEN.cu [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def main(rep, cubin, src, top=25):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    line = None
    loc = {}
    for ln in dis.splitlines():
        m = re.search(r'//## File "(.*)", line (\d+)', ln)
        if m:
            line = int(m.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and line is not None:
            loc[int(m.group(1), 16)] = line
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, iw, ix = hdr.index("Address"), hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
    base = None
    tot = defaultdict(float)
    exc = defaultdict(float)
    for r in rows[2:]:
        a = int(r[ia], 16)
        base = a if base is None else base
        ln = loc.get(a - base)
        try:
            tot[ln] += float(r[iw])
            exc[ln] += float(r[ix])
        except ValueError:
            pass
    T = sum(tot.values())
    text = open(src).read().splitlines()
    print("total shared wavefronts %.4g, excessive %.4g" % (T, sum(exc.values())))
    for ln, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print("%6s %6.2f%% excess %6.2f%%  %s" % (ln, 100 * v / T, 100 * exc[ln] / T,
                                                 text[ln - 1].strip()[:90] if ln else "?"))


if __name__ == "__main__":
    main(*sys.argv[1:4], *(int(a) for a in sys.argv[4:5]))
