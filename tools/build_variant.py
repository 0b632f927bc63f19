"""Build a variant of libgsicp.so with extra nvcc flags (A/B experiments on the GPU box):
python tools/build_variant.py NAME [-DFLAG=V ...]  ->  paper_2403_12550_b200/variants/libgsicp_NAME.so
(tools/gpu_abv.sh swaps the variants in before each bench run)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_12550_b200 import _build as b  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(b.HERE, "variants")
    obj_dir = os.path.join(out_dir, "obj_" + name)
    os.makedirs(obj_dir, exist_ok=True)
    nv = b.nvcc()

    def one(s):
        obj = os.path.join(obj_dir, s.replace(".cu", ".o"))
        r = subprocess.run([nv, *b.FLAGS, *extra, "-c", os.path.join(b.CSRC, s), "-o", obj], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, b.SOURCES))
    lib = os.path.join(out_dir, f"libgsicp_{name}.so")
    subprocess.run([nv, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-o", lib, *objs],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
