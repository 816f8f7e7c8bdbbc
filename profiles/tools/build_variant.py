"""Build an A/B variant of libfractime_b200.so with extra nvcc flags (e.g. -DFT_NO_TWQ):

    python profiles/tools/build_variant.py NAME [nvcc flags ...]

-> paper_1710_11593_b200/_variants/NAME.so; run with FT_LIB_VARIANT=<that path>."""
import subprocess, sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1710_11593_b200 import build as B

name, flags = sys.argv[1], sys.argv[2:]
out = B.PKG / "_variants"; out.mkdir(exist_ok=True)
tmp = out / ("_obj_" + name); tmp.mkdir(exist_ok=True)


def cc(src):
    o = tmp / (src + ".o")
    cmd = [B.nvcc(), *B.ARCH, *B.COMMON, *B.EXTRA.get(src, []), *flags, "-c", str(B.CSRC / src), "-o", str(o)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, B.SOURCES))
lib = out / (name + ".so")
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart_static", "-lrt", "-ldl",
                "-lpthread"], check=True)
print(lib)
