"""Static SASS census of a kernel (local, no GPU): instruction mix of the largest loop.
usage: python scripts/sass_loop.py <mangled-name-substring>"""
import re, subprocess, sys
from collections import Counter
lib = "paper_2407_19097_b200/libnar_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
name = sys.argv[1]
blocks = re.split(r"\n\s+Function : ", out)
for b in blocks:
    if name in b.split("\n")[0]:
        lines = [l for l in b.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
        ins = []
        for l in lines:
            m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", l)
            if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
        # find backward branches -> loops
        loops = []
        for addr, txt in ins:
            m = re.search(r"BRA(?:\.\w+)* (?:!?U?P\d, )?0x([0-9a-f]+)", txt)
            if m and int(m.group(1), 16) < addr:
                loops.append((int(m.group(1), 16), addr))
        lo, hi = max(loops, key=lambda t: t[1] - t[0])
        body = [t for a, t in ins if lo <= a <= hi]
        ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
        print(b.split("\n")[0][:80], "loop", hex(lo), hex(hi), "instructions", len(body))
        for k, v in ops.most_common(30): print(f"{v:5d} {k}")
        break
