"""Summarise an ncu --csv launch list: per-kernel count, serialized time and SM-time.

SM-time = sm__cycles_active.sum / SM clock: the SM-seconds a kernel keeps busy, i.e. its cost
when many streams pack the GPU (divide by 148 for the fully-packed wall time)."""
import collections
import csv
import sys

NSM = 148


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    k = collections.OrderedDict()
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d['ID'], d['Kernel Name'])
        v = float(d['Metric Value'].replace(',', ''))
        u = d['Metric Unit']
        m = d['Metric Name']
        if m == 'gpu__time_duration.sum':
            v = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}[u] * v
        elif m == 'sm__cycles_elapsed.avg.per_second':
            v = {'hz': 1.0, 'khz': 1e3, 'Mhz': 1e6, 'mhz': 1e6, 'Ghz': 1e9, 'ghz': 1e9, 'cycle/second': 1.0,
                 'cycle/nsecond': 1e9, 'cycle/usecond': 1e6}.get(u, 1.0) * v
        k.setdefault(key, {})[m] = v
    return k


def main(path, top=25):
    k = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in k.items():
        n = name.split('(')[0].replace('(anonymous namespace)::', '')[:64]
        a = agg[n]
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0.0)
        if 'sm__cycles_active.sum' in m and m.get('sm__cycles_elapsed.avg.per_second'):
            a[2] += m['sm__cycles_active.sum'] / m['sm__cycles_elapsed.avg.per_second'] * 1e6 / NSM
    tot = sum(a[1] for a in agg.values())
    tsm = sum(a[2] for a in agg.values())
    print(f"kernels {sum(a[0] for a in agg.values())}  serialized {tot / 1e3:.3f} ms  "
          f"packed (SM-time/{NSM}) {tsm / 1e3:.3f} ms")
    print(f"{'serial ms':>10} {'packed ms':>10} {'n':>6} {'avg us':>8}  kernel")
    for n, (c, t, sm) in sorted(agg.items(), key=lambda x: -x[1][2] if tsm else -x[1][1])[:top]:
        print(f"{t / 1e3:10.3f} {sm / 1e3:10.3f} {c:6d} {t / c:8.2f}  {n}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
