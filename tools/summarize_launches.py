"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv`) of one solve step by kernel, and optionally write the
per-launch DRAM traffic of the bench's roofline kernels.

    python tools/summarize_launches.py profiles/r01_launches.csv [--traffic profiles/traffic.json] \
        > profiles/r01_launches.md

Stage mapping for --traffic (launch order inside a step is fixed by run_rsvd):
  jacobi     -> k_jacobi_blk
  cholinv    -> k_cholinv* (mean over the step's launches)
  assemble   -> the row-walk kernels (sum: one assembly)
  gemm_power -> mean over the step's power-product launches (gemm_tc_kernel<256, 1, 1>)
  gemm_apply -> k_apply_fused
"""
import collections
import csv
import json
import sys

UNITS = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "nsecond": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ii, ik, im = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name")
    iv, iu = hdr.index("Metric Value"), hdr.index("Metric Unit")
    ig, ib = hdr.index("Grid Size"), hdr.index("Block Size")
    launches = collections.OrderedDict()
    for r in data:
        lid = int(r[ii])
        name = r[ik].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        ent = launches.setdefault(lid, {"name": name, "grid": r[ig], "block": r[ib]})
        v = float(r[iv].replace(",", "")) * UNITS.get(r[iu], 1.0)
        if r[im] == "gpu__time_duration.sum":
            ent["us"] = v
        elif r[im].startswith("dram__bytes"):
            ent["dram"] = ent.get("dram", 0.0) + v
    return list(launches.values())


def main(argv):
    path = argv[0]
    traffic_out = argv[argv.index("--traffic") + 1] if "--traffic" in argv else None
    L = load(path)
    agg = collections.OrderedDict()
    tot = sum(x.get("us", 0.0) for x in L)
    have_dram = any("dram" in x for x in L)
    for x in L:
        a = agg.setdefault(x["name"], [0, 0.0, 0.0, x["grid"], x["block"]])
        a[0] += 1
        a[1] += x.get("us", 0.0)
        a[2] += x.get("dram", 0.0)
    print(f"# ncu launch list: {path}\n")
    print(f"{len(L)} launches, {tot:.1f} us total (cold-cache, serialised: compare shares, not absolutes)\n")
    if have_dram:
        print("| kernel | launches | total us | share | DRAM MB / launch | grid | block |")
        print("|---|---|---|---|---|---|---|")
    else:
        print("| kernel | launches | total us | share | grid | block |")
        print("|---|---|---|---|---|---|")
    for k, (n, us, dram, g, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        extra = f" {dram / n / 1e6:.1f} |" if have_dram else ""
        print(f"| {k} | {n} | {us:.1f} | {100 * us / tot:.1f}% |{extra} {g} | {b} |")
    if traffic_out and have_dram:
        def per_launch(pred):
            xs = [x["dram"] for x in L if pred(x["name"])]
            return sum(xs) / len(xs) if xs else None
        # power products: the 3xF16 twin kernel <256, 1, 1> (round 1: gemm_tf32x3); the first launch is Y0 = X Omega
        gemms = [x for x in L if x["name"].startswith("gemm_tf32x3") or x["name"].startswith("gemm_tc_kernel<256, 1, 1>")]
        asm = [x["dram"] for x in L if x["name"] in ("k_seg_sort", "k_assemble_rows", "k_assemble", "k_assemble_rows3")]
        traffic = {
            "jacobi": per_launch(lambda n: n.startswith("k_jacobi")),
            "cholinv": per_launch(lambda n: n.startswith("k_cholinv")),
            "assemble": sum(asm) if asm else None,
            "gemm_power": (sum(x["dram"] for x in gemms) / len(gemms)) if gemms else None,
            "gemm_apply": per_launch(lambda n: n.startswith("k_apply_fused")),
            "source": path + " (ncu dram__bytes_read.sum + dram__bytes_write.sum, one step, bytes per launch)",
        }
        json.dump(traffic, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
