"""Build an experimental libnmq variant: tools/build_variant.py NAME -DFLAG=V ...
-> paper_2305_02678_b200/variants/libnmq_NAME.so (select with NMQ_LIB=...)."""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_02678_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "paper_2305_02678_b200", "variants")
os.makedirs(out_dir, exist_ok=True)
saved_out, saved_obj = B.OUT, B.OBJ
B.OUT = os.path.join(out_dir, f"libnmq_{name}.so")
B.OBJ = os.path.join(ROOT, "build", f"nmq_{name}")
B.build(extra=flags)
print(B.OUT)
