"""Parse the globaltimer stamps of a GS_PROF_TL build (find CTAs: F lines,
update lead: U lines) and print the per-batch critical path of the
find -> update chain.  Usage: python tools/timeline.py <log>"""
import collections
import sys

OFF = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # batch number of find launch 0
F = collections.defaultdict(list)
U = {}
for line in open(sys.argv[1]):
    p = line.split()
    if p and p[0] == "F":
        seq, blk, sm = map(int, p[1:4])
        F[seq].append(list(map(int, p[4:10])))
    elif p and p[0] == "U":
        b, sm, t0, t1, t2, win = map(int, p[1:7])
        U[b] = (t0, t1, t2, win)
for seq in sorted(F):
    rows = F[seq]
    e0 = min(r[0] for r in rows)  # first CTA resident
    w1 = min(r[1] for r in rows)  # first CTA past griddepcontrol.wait
    w1max = max(r[1] for r in rows)
    end = max(r[5] for r in rows)
    ph = [sorted(r[k] - r[k - 1] for r in rows) for k in range(2, 6)]
    med = [p[len(p) // 2] / 1e3 for p in ph]
    mx = [p[-1] / 1e3 for p in ph]
    b = seq + OFF  # find launch s feeds update batch s + OFF
    prev = U.get(b - 1)
    cur = U.get(b)
    s = f"find {seq}: ctas={len(rows)} wait-spread={(w1max - w1) / 1e3:.2f}us run={(end - w1) / 1e3:.2f}us " \
        f"phases med stage/pass1/screen/exact+store = " + "/".join(f"{x:.2f}" for x in med) + \
        " max " + "/".join(f"{x:.2f}" for x in mx)
    if prev:
        s += f" | prev update end -> find wait released {(w1 - prev[2]) / 1e3:.2f}us"
    if cur:
        s += f" | find end -> update wait released {(cur[1] - end) / 1e3:.2f}us, update run " \
             f"{(cur[2] - cur[1]) / 1e3:.2f}us (resident {(cur[1] - cur[0]) / 1e3:.2f}us early, windows {cur[3]})"
    print(s)
