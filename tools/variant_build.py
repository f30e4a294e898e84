"""Build A/B variants of one libsdp source file into tools/_variants/<name>/libsdp.so
(the other objects come from the current in-tree build).  Probe-only.

    python tools/variant_build.py NAME SRC.cu [SRC_REPLACEMENT_FILE.cu]
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2507_09029_b200 import build as B  # noqa: E402


def main():
    name, src = sys.argv[1], Path(sys.argv[2])
    out = ROOT / "tools" / "_variants" / name
    out.mkdir(parents=True, exist_ok=True)
    stem = Path(sys.argv[3]).stem if len(sys.argv) > 3 else src.stem
    obj = out / (stem + ".o")
    # the variant source lives outside csrc/ (so the in-tree build never sees
    # it); csrc/ on the include path resolves its headers
    tmp = out / src.name
    tmp.write_text(src.read_text())
    r = subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, "-I", str(B.CSRC), "-c", str(tmp), "-o", str(obj)],
                       capture_output=True, text=True)
    (out / "ptxas.log").write_text(r.stderr)
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    objs = [str(obj)] + [str(o) for o in sorted((B.LIBDIR / "obj").glob("*.o")) if o.stem != stem]
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out / "libsdp.so"), *objs, "-cudart", "static"],
                   check=True)
    print(out / "libsdp.so")


if __name__ == "__main__":
    main()
