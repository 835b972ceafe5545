"""Kernel shares and rns_kernel DRAM traffic of one timed bench step, from the
ncu launch list of tools/profile_bench_launches.sh (gpu__time_duration +
dram bytes per launch).  Writes the RNS entries of profiles/traffic.json and
prints the per-kernel shares.

  python tools/traffic_from_launches.py profiles/round2/launches_bench_r2.csv
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
        "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def launches(path):
    hdr, out = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = out.setdefault(d["ID"], {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "")})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]]
    return list(out.values())


def main():
    src = sys.argv[1]
    ls = launches(src)
    idx = [i for i, e in enumerate(ls) if e["kernel"].endswith("rns_kernel")]
    last = idx[-33:]  # the timed step: 33 products, packs before each rns_kernel, CRT after
    step = ls[last[0] - 2:last[-1] + 2]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for e in step:
        tot[e["kernel"]] += e["gpu__time_duration.sum"]
        cnt[e["kernel"]] += 1
    T = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print("%-45s %3d launches %8.2f ms %5.1f%%" % (k, cnt[k], v / 1e6, 100 * v / T))
    dram = [ls[i]["dram__bytes_read.sum"] + ls[i]["dram__bytes_write.sum"] for i in last]
    # algorithmic bytes per launch: A and B residues + parked residues, n moduli at 8192^3
    sys.path.insert(0, ROOT)
    import paper_2601_07508_b200 as F
    alg = []
    for b in range(20, 53):
        n = F.rns_plan(F.prev_prime(1 << b), 8192)["n"]
        alg.append(3.0 * n * 8192 * 8192)
    avg, aavg = sum(dram) / len(dram), sum(alg) / len(alg)
    print("rns_kernel DRAM per launch: sweep average %.2f GB (algorithmic %.2f GB, %.2fx)" % (avg / 1e9, aavg / 1e9,
                                                                                          avg / aavg))
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    db = json.load(open(tj))
    rel = os.path.relpath(src, ROOT)
    entry = {
        "kernel": "rns_kernel over the 8192^3 sweep (20..52 bits, 7..15 byte moduli; CTA pairs, M256 N256, 256-byte "
                  "k stages, flat pass order)",
        "dram_bytes_per_launch": round(avg),
        "algorithmic_bytes_per_launch": round(aavg),
        "per_bits_dram_bytes": {str(b): round(x) for b, x in zip(range(20, 53), dram)},
        "note": "dram__bytes_read.sum + dram__bytes_write.sum of each of the 33 rns_kernel launches of one timed step "
                "of the default bench command under ncu (%s), averaged per launch like roofline.achieved. "
                "Algorithmic = A residues (n*m*k) + B residues (n*k*n) + parked residues (n*m*n)." % rel,
        "source": rel,
    }
    db["rns"] = dict(entry)
    db["auto"] = dict(entry)
    json.dump(db, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
