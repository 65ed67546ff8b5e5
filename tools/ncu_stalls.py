"""Per-SASS-instruction stall samples of one reason from an ncu report (--import-source on):
python tools/ncu_stalls.py REPORT REASON [N]   (REASON e.g. stall_long_sb) — development aid."""
import csv, subprocess, sys
rep, reason = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
hdr, cur, rows = None, None, []
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == 'Line No':
        hdr = r
        col = hdr.index(reason)
        continue
    if not hdr:
        continue
    if r[0].isdigit():
        cur = r[0]
    elif r[0] == '' and len(r) > col:
        try:
            v = int(r[col] or 0)
        except ValueError:
            continue
        if v:
            rows.append((v, cur, r[2], r[3].strip()[:70]))
tot = sum(x[0] for x in rows) or 1
print(f"{reason}: total {tot}")
for v, line, addr, sass in sorted(rows, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  line {line:>5} {addr[-5:]}  {sass}")
