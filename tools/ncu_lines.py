"""Per-source-line hotspots of an ncu report (--import-source on, -lineinfo):
warp-stall samples and excess shared-memory wavefronts by CUDA line
(development aid): python tools/ncu_lines.py REPORT [N]"""
import csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows, fname, hdr = [], None, None
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr and r[0].isdigit():  # CUDA line rows (SASS rows under them have an empty first column)
        try:
            s = int(r[4] or 0)
            ex = int(r[hdr.index('L1 Wavefronts Shared Excessive')] or 0)
        except (ValueError, IndexError):
            continue
        if s or ex:
            rows.append((s, ex, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(r[0] for r in rows) or 1
print(f"total stall samples {tot}")
for s, ex, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  excess_shared_wavefronts {ex:>11}  {loc:24s} {src}")
print("top excess shared wavefronts:")
for s, ex, loc, src in sorted(rows, key=lambda r: -r[1])[:8]:
    print(f"  {ex:>11}  {loc:24s} {src}")
