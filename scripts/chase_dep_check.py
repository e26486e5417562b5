"""Exhaustive footprint check of the carried-block bulge chase (stage2_chase.cu, ch2):
block k of sweep s may be loaded once sweep s-1 finished ops <= k+3 and stored their
non-carried blocks (lag K = 4); K = 3 is shown to fail.  Development aid."""
import sys, itertools
def ops(s, n, b):
    """list of ops of sweep s: dict(kind, rows, cols (logical footprint), load(global read set), store(global write set at op end), carry_out)"""
    out = []
    e0 = min(s + 1 + b, n)
    rows = range(s, e0); cols = range(s + 1, e0)
    fp = {(r, c) for r in rows for c in cols}
    carry = {(r, c) for r in range(s + 1, e0) for c in cols}
    out.append(dict(i=0, fp=fp, load=set(fp), store=fp - carry, carry=carry))
    r0 = s + 1
    while r0 < n:
        rE = min(r0 + b, n); cE = min(r0 + 2 * b, n)
        fp = {(r, c) for r in range(r0, rE) for c in range(r0, cE)}
        D = {(r, c) for r in range(r0, rE) for c in range(r0, min(r0 + b, n))}
        E = fp - D
        out.append(dict(i=len(out), fp=fp, load=E, store=D, carry=E))
        if r0 + b >= n: break
        fp = {(r, c) for r in range(r0, cE) for c in range(r0 + b, cE)}
        P = {(r, c) for r in range(r0, r0 + b) for c in range(r0 + b, cE)}
        Q = fp - P
        out.append(dict(i=len(out), fp=fp, load=Q, store=P, carry=Q))
        r0 += b
    return out

def check(n, b, K):
    S = n - 2
    allops = [ops(s, n, b) for s in range(S)]
    bad = 0
    for s in range(1, S):
        for op in allops[s]:
            i = op['i']
            for k in range(1, s + 1):
                prev = allops[s - k]
                need = i + K * k   # ops of s-k completed (0..need-1) when (s,i) starts
                # (a) later ops of s-k must not touch our logical footprint
                for j in range(need, len(prev)):
                    if prev[j]['fp'] & op['fp']:
                        bad += 1
                        if bad < 5: print(f"n={n} b={b} K={K}: overlap ({s},{i}) with ({s-k},{j})")
                # (b) anything we load from global that s-k modified must be written back:
                #     element last touched by op j of s-k; if carried by j, written at j+1 (must be < need)
                for j in range(min(need, len(prev))):
                    pj = prev[j]
                    if pj['carry'] & op['load'] and j + 1 >= need:
                        # is it also touched later (j+1 writes back)? j+1 < need required
                        bad += 1
                        if bad < 5: print(f"n={n} b={b} K={K}: stale carried read ({s},{i}) <- ({s-k},{j})")
    return bad

for b in (2, 3, 4, 5, 8):
    for n in (3, 4, 7, 2 * b + 1, 4 * b, 4 * b + 3, 6 * b + 1):
        if n < 3: continue
        for K in (4, 5):
            r = check(n, b, K)
            print(f"b={b} n={n} K={K}: {'OK' if r == 0 else 'FAIL %d' % r}")
