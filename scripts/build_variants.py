"""Scratch: build tuning variants of libb200ipc.so (spmv.cu / pcg.cu recompiled with -D overrides).
usage: build_variants.py tag:KEY=VAL,KEY=VAL ...   -> scripts/probes/_bin/libb200ipc_<tag>.so"""
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2308_09400_b200 import _build
out = "scripts/probes/_bin"; os.makedirs(out, exist_ok=True)
_build.build()
for spec in sys.argv[1:]:
    tag, _, defs = spec.partition(":")
    dflags = ["-D" + d for d in defs.split(",") if d]
    objs = []
    for src in _build.SOURCES:
        obj = os.path.join(_build.OBJ, src.replace(".cu", ".o"))
        if src in os.environ.get("VARIANT_SOURCES", "spmv.cu,pcg.cu").split(","):
            obj = os.path.join(out, f"{tag}_{src.replace('.cu', '.o')}")
            subprocess.check_call([_build._nvcc()] + _build.NVCC_FLAGS + dflags + ["-c", os.path.join(_build.CSRC, src), "-o", obj])
        objs.append(obj)
    lib = os.path.join(out, f"libb200ipc_{tag}.so")
    subprocess.check_call([_build._nvcc(), "-shared", "-o", lib] + objs + ["-lcudart"])
    print(lib)
