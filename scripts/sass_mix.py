"""Static SASS opcode census of one kernel in libbnn.so (optionally an address range).
   python scripts/sass_mix.py <mangled-name-substring> [lo_hex hi_hex]"""
import collections
import re
import subprocess
import sys

so = "paper_2604_04736_b200/libbnn.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
sel = [f for f in funcs if sys.argv[1] in f.split("\n", 1)[0]]
for f in sel:
    name = f.split("\n", 1)[0]
    ins = [(int(a, 16), t) for a, t in re.findall(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", f)]
    if len(sys.argv) > 3:
        lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
        ins = [(a, t) for a, t in ins if lo <= a < hi]
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for a, t in ins)
    print(name[:100], "total", sum(c.values()))
    print("  " + "  ".join(f"{k}:{v}" for k, v in c.most_common(30)))
