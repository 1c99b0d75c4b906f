"""Compile the generated SSA kernels for C1..C5 with NVRTC (the same library and
options jit.cpp uses on the GPU box, so the cubin is the binary that runs) on a
machine without a GPU: catches codegen errors and reports registers / spills /
static SASS size.  Writes build/gen/<cfg>_v<variant>.cu and .cubin.

  python scripts/check_codegen.py [C1 C2 ...]       (SMC_TILE_WIDTH, SMC_SW_S honoured)
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
import paper_0912_2551_b200 as smc  # noqa: E402

# keep in sync with jit.cpp
OPTS = [b"--gpu-architecture=sm_100a", b"--std=c++17", b"--fmad=false", b"-lineinfo",
        b"--extra-device-vectorization", b"-DNDEBUG", b"-Xptxas=-v"]


def nvrtc_cubin(src, name):
    lib = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
    prog = ctypes.c_void_p()
    assert lib.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), name.encode(), 0, None, None) == 0
    opts = (ctypes.c_char_p * len(OPTS))(*OPTS)
    rc = lib.nvrtcCompileProgram(prog, len(OPTS), opts)
    n = ctypes.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    if rc != 0:
        raise SystemExit("NVRTC failed for %s:\n%s" % (name, log.value.decode()[:4000]))
    lib.nvrtcGetCUBINSize(prog, ctypes.byref(n))
    buf = ctypes.create_string_buffer(n.value)
    lib.nvrtcGetCUBIN(prog, buf)
    lib.nvrtcDestroyProgram(ctypes.byref(prog))
    return buf.raw, log.value.decode()


def main(names):
    out = os.path.join(ROOT, "build", "gen")
    os.makedirs(out, exist_ok=True)
    for name in names:
        cfg = workloads.get(name)
        small = len(cfg["species"]) <= 32 and len(cfg["reactions"]) <= 32
        for variant in ([1, 2, 4] if small else [2, 4, 5]):
            m = smc.Model.from_config(cfg)
            try:
                m.set_variant(variant)
            except smc.SmcError:
                continue
            p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
            src = m.kernel_source(p)
            path = os.path.join(out, "%s_v%d.cu" % (name, variant))
            with open(path, "w") as fh:
                fh.write(src)
            cubin, log = nvrtc_cubin(src, path)
            with open(path[:-3] + ".cubin", "wb") as fh:
                fh.write(cubin)
            sass = subprocess.run(["cuobjdump", "-sass", path[:-3] + ".cubin"], capture_output=True, text=True).stdout
            n_inst = sum(1 for ln in sass.splitlines() if ln.strip().startswith("/*") and "*/" in ln.strip()[:10])
            info = [ln.strip() for ln in log.splitlines() if "registers" in ln or "spill" in ln]
            print(name, "v%d" % variant, "sass=%d" % n_inst, " | ".join(info))


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
