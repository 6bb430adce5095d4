"""Where the host link idles: reads a raw span dump (bench.py TC_DUMP_TIMELINE=FILE, spans of one sync interval, e.g.
with TC_DIAG_RETIRE=1 the whole retire-each diagnostic loop) and reports, per DMA direction, busy time, the union and
intersection of the two directions, and the idle gaps between consecutive DMA runs with what the stream ran in them.

    python tools/timeline_gaps.py gpurun_out/timeline.json
"""
import json
import sys


def union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def length(iv):
    return sum(b - a for a, b in iv)


def intersect(x, y):
    i = j = 0
    out = []
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append([a, b])
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


def main(path):
    spans = json.load(open(path))
    by_sync = {}
    for s in spans:
        by_sync.setdefault(s[0], []).append(s)
    sync = max(by_sync, key=lambda k: len(by_sync[k]))
    sp = by_sync[sync]
    t_end = max(s[3] for s in sp)
    d2h = union([[s[2], s[3]] for s in sp if s[1] == "memcpy_d2h"])
    h2d = union([[s[2], s[3]] for s in sp if s[1] == "memcpy_h2d"])
    both = intersect(d2h, h2d)
    either = union(d2h + h2d)
    print(f"sync {sync}: {len(sp)} spans over {t_end:.3f} ms")
    print(f"  d2h busy {length(d2h):.3f} ms ({length(d2h) / t_end:.3f}), h2d busy {length(h2d):.3f} ms "
          f"({length(h2d) / t_end:.3f}), both {length(both):.3f}, either {length(either):.3f}, neither "
          f"{t_end - length(either):.3f}")
    nb = {"memcpy_d2h": 0, "memcpy_h2d": 0}
    for s in sp:
        if s[1] in nb:
            nb[s[1]] += s[4]
    for k, iv in (("memcpy_d2h", d2h), ("memcpy_h2d", h2d)):
        gaps = [(iv[i][1], iv[i + 1][0]) for i in range(len(iv) - 1)]
        g = sorted((b - a for a, b in gaps), reverse=True)
        print(f"  {k}: {len(iv)} runs, {nb[k] / 1e9 / (length(iv) * 1e-3):.1f} GB/s while busy, gaps total "
              f"{sum(g):.3f} ms, largest {[round(x, 3) for x in g[:6]]}, median {g[len(g) // 2] if g else 0:.3f}")
        for a, b in gaps[:8]:
            inside = sorted({s[1] for s in sp if s[2] < b and s[3] > a and s[1] != k})
            print(f"     gap {a:.3f}-{b:.3f} ({b - a:.3f} ms): {inside}")


if __name__ == "__main__":
    main(sys.argv[1])
