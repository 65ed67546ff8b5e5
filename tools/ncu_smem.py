"""Shared-memory wavefronts (actual / ideal) per CUDA source line from the SASS rows of an
ncu source page (--import-source on) — development aid: python tools/ncu_smem.py REPORT [UNITS]"""
import csv, subprocess, sys
rep = sys.argv[1]
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
hdr, cur, agg, src, fname = None, None, {}, {}, None
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        iw, ii = hdr.index('L1 Wavefronts Shared'), hdr.index('L1 Wavefronts Shared Ideal')
        continue
    if not hdr:
        continue
    if r[0].isdigit():
        cur = f"{fname}:{r[0]}"
        src[cur] = r[1].strip()[:70]
    elif r[0] == '' and cur and len(r) > iw:
        try:
            w, i = int(r[iw] or 0), int(r[ii] or 0)
        except ValueError:
            continue
        if w:
            a = agg.setdefault(cur, [0, 0, set()])
            a[0] += w
            a[1] += i
            a[2].add(r[3].strip().split(' ')[0])
tw = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"total wavefronts {tw} ({tw / per:.1f} per unit), ideal {ti} ({ti / per:.1f})")
for k, (w, i, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{w / per:8.1f} {i / per:8.1f}  {k:24s} {','.join(sorted(ops))[:30]:30s} {src.get(k, '')}")
