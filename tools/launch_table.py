"""Per-kernel table (time, DRAM bytes, GB/s) from an ncu --csv launch list that collected
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum."""
import collections
import csv
import sys


def main(path, top=20):
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
        key = (d['ID'], d['Kernel Name'].split('(')[0].replace('(anonymous namespace)::', '')[:56])
        k.setdefault(key, {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, n), m in k.items():
        a = agg[n]
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0.0) / 1e3
        a[2] += (m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)) / 1e6
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} kernels")
    print(f"{'us':>9} {'n':>4} {'avg us':>8} {'DRAM MB':>9} {'GB/s':>8}  kernel")
    for n, (c, t, mb) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:9.1f} {c:4d} {t / c:8.1f} {mb:9.2f} {mb / t * 1e3 if t else 0:8.1f}  {n}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
