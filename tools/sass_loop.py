"""Opcode histogram of a kernel's SASS (whole function and the hottest loop)."""
import collections
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for p in re.split(r'\n\s*Function : ', txt)[1:]:
    name = p.split('\n', 1)[0].strip()
    if not re.search(pat, name):
        continue
    ins = []
    for l in p.split('\n'):
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    # backward branches = loops; take the largest
    loops = []
    for addr, t in ins:
        m = re.search(r'BRA\s+(?:`\()?(?:\.L_x_\d+)?\)?\s*0x([0-9a-f]+)', t)
        if m and 'BRA' in t:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                loops.append((addr - tgt, tgt, addr))
    print(name, 'total', len(ins))
    for size, a, b in sorted(loops, reverse=True)[:2]:
        c = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', t).split()[0].split('.')[0] for x, t in ins if a <= x <= b)
        print(f'  loop {a:#x}-{b:#x}: {sum(c.values())} instr', c.most_common(25))
