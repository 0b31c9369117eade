"""Build an experimental libplgpu.so variant with extra nvcc defines into
paper_1407_2343_b200/lib/var_<tag>/libplgpu.so (use with PLGPU_LIB=...).

    python tools/build_variant.py <tag> -DPLGPU_PRESCALE=1 [...]
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_2343_b200 import build as B  # noqa: E402


def main():
    tag, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join("/tmp", f"plgpu_var_{tag}")
    os.makedirs(out, exist_ok=True)
    units = [(os.path.join(B.CSRC, "plgpu.cu"), os.path.join(out, "plgpu.o"))]
    radii = [int(r) for r in os.environ["RADII"].split(",")] if os.environ.get("RADII") else B.WALK_RADII
    units += [(B._gen_inst(r), os.path.join(out, f"inst_S{r}.o")) for r in B.WALK_RADII]
    # radii not rebuilt (RADII=10,15,25 for quick experiments) reuse the main build's objects
    units = [(s, o if any(s.endswith(f"inst_S{r}.cu") for r in radii) or s.endswith("plgpu.cu")
              else os.path.join(B.BUILD, "obj", os.path.basename(o))) for s, o in units]

    def one(so):
        B._run([B.NVCC] + B.NVFLAGS + extra + ["-c", so[0], "-o", so[1]])

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        list(ex.map(one, [u for u in units if u[1].startswith(out)]))
    libdir = os.path.join(B.LIB, f"var_{tag}")
    os.makedirs(libdir, exist_ok=True)
    lib = os.path.join(libdir, "libplgpu.so")
    B._run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + [o for _, o in units])
    print(lib)


if __name__ == "__main__":
    main()
