"""Write profiles/traffic_<tag>.json: DRAM bytes (read + write) per launch of the SSA
kernel from ncu --set full captures, for bench.py's roofline.traffic field.
  python scripts/ncu_traffic.py TAG WORKLOAD=rep.ncu-rep[:note] ...
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(r[i]) * scale[units[i]]
    def f(m):
        return float(r[hdr.index(m)]) if m in hdr and r[hdr.index(m)] not in ("", "n/a") else None
    wf, wfi = f("memory_l1_wavefronts_shared"), f("memory_l1_wavefronts_shared_ideal")
    return {"kernel": r[hdr.index("Kernel Name")], "dram_bytes_per_launch": tot,
            "duration_ns": float(r[hdr.index("gpu__time_duration.sum")]) *
                           {"s": 1e9, "ms": 1e6, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(
                               units[hdr.index("gpu__time_duration.sum")], 1.0),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "smem_wavefront_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "smem_wavefront_excess": (wf / wfi) if wf and wfi else None}


def main(tag, specs):
    out = {}
    for s in specs:
        w, rest = s.split("=", 1)
        rep, _, note = rest.partition(":")
        d = dram(rep)
        d["capture"] = os.path.basename(rep)
        d["note"] = note
        out[w] = d
    path = os.path.join(ROOT, "profiles", "traffic_%s.json" % tag)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
