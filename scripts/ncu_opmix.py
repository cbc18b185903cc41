"""Opcode mix and stall samples of one kernel from an `ncu --page source --csv` export.
usage: python scripts/ncu_opmix.py file.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]; data = rows[hi + 1:]
iS = hdr.index('Source'); iE = hdr.index('Instructions Executed'); iSamp = hdr.index('# Samples')
ops = collections.Counter(); samp = collections.Counter(); tot = 0
for r in data:
    if len(r) <= iE or not r[iE].isdigit(): continue
    toks = r[iS].strip().split()
    op = toks[0] if not toks[0].startswith('@') else toks[1]
    op = '.'.join(op.split('.')[:2]) if op.startswith(('LDS', 'STG', 'LDG', 'STS')) else op.split('.')[0]
    n = int(r[iE]); ops[op] += n; tot += n; samp[op] += int(r[iSamp])
print('total warp instructions', tot, 'samples', sum(samp.values()))
for op, n in ops.most_common(30):
    print(f"{op:12s} {n:10d} {100*n/tot:5.1f}%  samples {samp[op]:6d} {100*samp[op]/max(1,sum(samp.values())):5.1f}%")
st = [(h, i) for i, h in enumerate(hdr) if h.startswith('stall_')]
tots = {h: sum(int(r[i]) for r in data if len(r) > i and r[i].isdigit()) for h, i in st}
print({h: v for h, v in sorted(tots.items(), key=lambda kv: -kv[1]) if v})
