"""List the source lines of local-memory (spill) accesses in one kernel of a cubin:
    python tools/spill_lines.py file.cubin kernel_substring"""
import re
import subprocess
import sys

cub, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.split("\n")
inside, cur = False, None
for l in out:
    if ".text." in l and ("section" in l or l.strip().startswith(".text")):
        inside = name in l
    if not inside:
        continue
    m = re.search(r'## File ".*?/([\w.]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    if re.search(r"\b(STL|LDL)\b", l):
        print(cur, l.strip()[:90])
