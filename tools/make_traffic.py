"""profiles/ncu_traffic.json: DRAM bytes (read + write) per launch for each op class, from an
ncu launch list with dram__bytes_read.sum / dram__bytes_write.sum (cold-cache: ncu flushes the
caches between kernels, so these are upper bounds on the warm-L2 traffic of the bench)."""
import collections
import csv
import json
import sys

CLASSES = [("jacobi", "jacobi"), ("potrf", "cholesky"), ("chol_fused", "cholesky"), ("gemm_kernel", "gemm"),
           ("splitk_reduce", "gemm"),
           ("spmm", "spmm"), ("seg_reduce", "spmm"), ("empty_rows", "spmm"), ("sddmm", "sddmm")]


def main(path, out):
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
        k.setdefault((d['ID'], d['Kernel Name']), {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for (_, name), m in k.items():
        for key, cls in CLASSES:
            if key in name:
                a = agg[cls]
                if key in ("gemm_kernel", "jacobi", "potrf", "chol_fused", "spmm", "sddmm"):
                    a[0] += 1
                a[1] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
                break
    res = {c: round(b / max(n, 1)) for c, (n, b) in agg.items()}
    res["_source"] = f"{path} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, cold cache, per main-kernel launch)"
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])
