"""Print the SASS of the kernels in a .so whose mangled name contains a substring.

    python tools/sass_of.py paper_2305_04966_b200/libnacc.so march_fused_kernelILb0ELb1ELb1 [--stats]
"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, keep = None, []
for ln in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", ln)
    if m:
        cur = m.group(1)
    if cur and pat in cur:
        keep.append(ln)
if "--stats" in sys.argv:
    ins = [l for l in keep if re.match(r"\s*/\*[0-9a-f]{4}\*/", l)]
    print(len(ins), "instructions;", sum("STL" in l or "LDL" in l for l in ins), "local ld/st")
else:
    print("\n".join(keep))
