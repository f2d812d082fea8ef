"""Per-kernel DRAM bytes (MB) and time from an ncu --csv launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum), averaged over the launches of each kernel.

    python profiles/dram_per_kernel.py launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    m = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            m[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    tot_r = tot_w = tot_t = 0.0
    for k, v in m.items():
        rd = sum(v["dram__bytes_read.sum"]) / len(v["dram__bytes_read.sum"]) / 1e6
        wr = sum(v["dram__bytes_write.sum"]) / len(v["dram__bytes_write.sum"]) / 1e6
        t = sum(v["gpu__time_duration.sum"]) / len(v["gpu__time_duration.sum"]) / 1e3
        tot_r, tot_w, tot_t = tot_r + rd, tot_w + wr, tot_t + t
        print(f"  {k:34s} {t:9.1f} us   DRAM rd {rd:8.1f} MB  wr {wr:8.1f} MB")
    print(f"  {'per iteration':34s} {tot_t:9.1f} us   DRAM rd {tot_r:8.1f} MB  wr {tot_w:8.1f} MB  total {tot_r + tot_w:.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1])
