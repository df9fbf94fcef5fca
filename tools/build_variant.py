"""Build an A/B variant of the C-ABI library with extra nvcc defines:
    python tools/build_variant.py OUT.so kr_sweep_f32.cu -DKR_SWEEP_PACKED_MINB=3 ...
Recompiles the named translation units with the extra flags and links them with
the main build's other objects (run `python -m paper_2605_11381_b200.build_lib` first)."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_11381_b200 import build_lib as bl  # noqa: E402

out = Path(sys.argv[1]).resolve()
srcs = [a for a in sys.argv[2:] if not a.startswith("-")]
flags = [a for a in sys.argv[2:] if a.startswith("-")]
bl.build()
tag = out.stem
objs = []
for src in bl.SOURCES:
    obj = bl.OBJ / (Path(src).stem + ".o")
    if src in srcs:
        obj = bl.OBJ / f"{Path(src).stem}.{tag}.o"
        subprocess.run([bl.nvcc(), *bl.NVCC_FLAGS, *flags, "-I", str(bl.INCLUDE), "-c",
                        str(bl.CSRC / src), "-o", str(obj)], check=True)
    objs.append(str(obj))
subprocess.run([bl.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                "-o", str(out), "-lcudart"], check=True)
print(out)
