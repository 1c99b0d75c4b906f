"""Cross-compile the generated SSA kernels for C1..C5 with nvcc (sm_100a) on a
machine without a GPU: catches codegen errors and shows registers / spills /
shared memory (-Xptxas -v).  Writes build/gen/<cfg>.cu and .cubin."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
import paper_0912_2551_b200 as smc  # noqa: E402


def main(names):
    out = os.path.join(ROOT, "build", "gen")
    os.makedirs(out, exist_ok=True)
    for name in names:
        cfg = workloads.get(name)
        for variant in ([1, 2] if len(cfg["species"]) <= 32 and len(cfg["reactions"]) <= 32 else [2]):
            m = smc.Model.from_config(cfg)
            m.set_variant(variant)
            p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
            src = m.kernel_source(p)
            path = os.path.join(out, "%s_v%d.cu" % (name, variant))
            with open(path, "w") as fh:
                fh.write(src)
            cmd = ["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "--fmad=false",
                   "-lineinfo", "-Xptxas", "-v", "-o", path[:-3] + ".cubin", path]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                print(r.stderr)
                raise SystemExit("codegen check failed for %s variant %d" % (name, variant))
            info = [ln.strip() for ln in r.stderr.splitlines() if "registers" in ln or "spill" in ln]
            print(name, "v%d" % variant, " | ".join(info))


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
