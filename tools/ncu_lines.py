"""Per-source-line instruction and stall shares of an ncu report (top N)."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
cur, agg = None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0].isdigit() and len(r) > 7 and r[2] == '-':
        try:
            agg.append((int(r[7]), int(r[4]), cur, int(r[0]), r[1][:90]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
tots = sum(a[1] for a in agg) or 1
print('total warp instructions', tot, 'stall samples', tots)
for a in sorted(agg, reverse=True)[:top]:
    print(f"{a[0] / tot * 100:5.1f}% inst {a[1] / tots * 100:5.1f}% stall  {a[2]}:{a[3]}  {a[4]}")
byf = collections.Counter()
for a in agg:
    byf[a[2]] += a[0]
print({k: round(v / tot, 3) for k, v in byf.items()})
