"""Parse SK_CS_PROF printf lines from k_lanczos_cols (one launch, side 0)."""
import sys, collections
W = collections.defaultdict(list); E = {}; L = {}; F = {}
for line in open(sys.argv[1]):
    t = line.split()
    if not t: continue
    if t[0] == "CSW": W[int(t[2])].append(tuple(int(x) for x in t[3:]))
    elif t[0] == "CSE": E[int(t[1])] = (int(t[2]), int(t[3]))
    elif t[0] == "CSL": L[int(t[1])] = (int(t[2]), int(t[3]))
    elif t[0] == "CSF": F[int(t[1])] = (int(t[2]), int(t[3]))
if E:
    t0 = min(v[0] for v in E.values())
    st = sorted(v[0] - t0 for v in E.values()); en = sorted(v[1] - t0 for v in E.values())
    print(f"CTAs {len(E)}: entry spread {st[0]}..{st[-1]} ns; loop end {en[0]}..{en[-1]} ns (median {en[len(en)//2]})")
    if L: print("line-node tails end:", sorted(v[1] - t0 for v in L.values()))
    if F: print("final:", [(v[0] - t0, v[1] - t0) for v in F.values()])
for w, v in sorted(W.items()):
    n = len(v); lines = sum(x[0] for x in v) / n
    print(f"warp {w:2d}: n={n} lines={lines:.0f} prologue={sum(x[1] for x in v)/n:.0f} cyc loop={sum(x[2] for x in v)/n:.0f} cyc work={sum(x[3] for x in v)/n:.0f} cyc")
