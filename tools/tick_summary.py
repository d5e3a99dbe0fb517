"""Summarises tools/tick_profile.py output on stdin: median / mean / max device µs, and the
mean over the heavy ticks (swing >= 1.5)."""
import statistics
import sys

rows = [(float(t[3]), float(t[5])) for t in (ln.split() for ln in sys.stdin)
        if len(t) > 5 and t[0] == "tick" and int(t[1]) > 0]
dev = [d for _, d in rows]
heavy = [d for s, d in rows if s >= 1.5]
print(f"median {statistics.median(dev):.1f} mean {statistics.mean(dev):.1f} max {max(dev):.1f} "
      f"heavy-mean {statistics.mean(heavy):.1f} (n={len(dev)})")
