"""List local-memory spill instructions (STL/LDL) of one kernel with their
source lines:  python tools/spills.py file.cubin SUBSTRING_OF_KERNEL_NAME"""
import re
import subprocess
import sys

cubin, key = sys.argv[1], sys.argv[2]
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.split("\n")
fn, loc = None, ""
for l in dis:
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
    if "//## File" in l:
        loc = l.split("//## File")[1].strip().replace('"/root/repo/paper_2305_02678_b200/csrc/', "")
    if fn and key in fn and re.search(r"\b(STL|LDL|CALL)\b", l):
        print(f"{loc[:48]:48s} | {l.strip()[:64]}")
