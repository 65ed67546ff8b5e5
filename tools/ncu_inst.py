"""Warp-level instructions executed per CUDA source line and per SASS opcode of an
ncu report (--import-source on, -lineinfo) — where a kernel's issue slots go
(development aid): python tools/ncu_inst.py REPORT [N] [--per UNITS]"""
import csv, re, subprocess, sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
per = float(sys.argv[sys.argv.index('--per') + 1]) if '--per' in sys.argv else 1.0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
lines, ops, fname, hdr, cur = Counter(), Counter(), None, None, None
src = {}
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        ie = hdr.index('Instructions Executed')
        continue
    if not hdr:
        continue
    if r[0].isdigit():
        cur = f"{fname}:{r[0]}"
        src[cur] = r[1].strip()[:80]
    elif r[0] == '' and len(r) > ie and cur:
        try:
            v = int(r[ie] or 0)
        except ValueError:
            continue
        sass = r[3].strip()
        op = re.sub(r'^@!?U?P\w+\s+', '', sass).split(' ')[0]
        lines[cur] += v
        ops[op] += v
tot = sum(lines.values()) or 1
print(f"total warp instructions {tot} ({tot / per:.1f} per unit)")
for loc, v in lines.most_common(n):
    print(f"{100 * v / tot:5.1f}% {v / per:9.1f}  {loc:26s} {src.get(loc, '')}")
print("by opcode:")
for op, v in ops.most_common(n):
    print(f"{100 * v / tot:5.1f}% {v / per:9.1f}  {op}")
