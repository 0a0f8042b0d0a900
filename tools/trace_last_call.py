"""Per-kernel busy time and span of the LAST call in an HSIM_TRACE log (calls end at k_merge)."""
import collections
import sys

L = [l.split() for l in open(sys.argv[1]) if l.startswith("TRACE")]
ends = [k for k, t in enumerate(L) if t[1] == "k_merge"]
a = ends[-2] + 1 if len(ends) > 1 else 0
last = L[a:ends[-1] + 1]
dur, cnt = collections.defaultdict(float), collections.Counter()
for t in last:
    dur[t[1]] += float(t[-1])
    cnt[t[1]] += 1
st, en = min(float(t[-3]) for t in last), max(float(t[-2]) for t in last)
print(f"{sys.argv[1]}: span {en - st:.1f} us, {len(last)} launches")
for k in sorted(dur, key=lambda k: -dur[k]):
    print(f"  {k:16s} x{cnt[k]:3d} {dur[k]:9.1f} us")
