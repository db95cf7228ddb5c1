"""Summarise the TRD_TRACE printout (per-CTA clock64 deltas of one column step
of trd_reduce_kernel at j = n/2): mean / max over the CTAs of each launch."""
import re
import statistics as st
import sys

rows = []
for l in open(sys.argv[1]):
    m = re.match(r'trd g=(\d+) j=(\d+): matvec (\-?\d+) upd (\-?\d+) xchg (\-?\d+) bar (\-?\d+) w (\-?\d+) refl (\-?\d+) total (\-?\d+) startns (\-?\d+)', l)
    if m:
        rows.append(tuple(int(x) for x in m.groups()))
G = int(sys.argv[2]) if len(sys.argv) > 2 else 148
names = ['matvec', 'upd', 'xchg', 'bar', 'w', 'refl', 'total', 'xchg_ns']
for L in range(0, len(rows), G):
    blk = rows[L:L + G]
    print(' '.join(f"{n} {st.mean(r[2 + i] for r in blk):.0f}/{max(r[2 + i] for r in blk)}" for i, n in enumerate(names)))
