"""profiles/dram_bytes.json from an ncu launch list of the bench command
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv): per-pass mean DRAM bytes, ncu duration and share of the pdgpu kernels.
usage: python profiles/dram_from_launches.py launches.csv [n batch] > profiles/dram_bytes.json
(n, batch: the lattice side and batch of the bench command; bench.py uses the
file only when they match its own workload)"""
import csv
import json
import sys

PASSES = [("k_rfft_rows", "K1_rfft_x"), ("k_spectral2d", "K3_spectral"), ("k_irfft_rows", "K5_irfft_x"),
          ("k_wrap", "K6w_wrap")]


def main(path, n=4096, batch=16):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        if "pdgpu" not in r[ki]:
            continue
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[ni]] = float(r[vi].replace(",", ""))
    tot_ms = sum(d.get("gpu__time_duration.sum", 0) for d in per.values()) / 1e6
    out = {"n": int(n), "batch": int(batch), "periodic": True,
           "source": f"ncu launch list {path} (bench command), mean over the launches of each pass",
           "dram_bytes_per_launch": {}, "ncu_ms_per_launch": {}, "share_of_pdgpu_kernels": {}}
    for key, name in PASSES:
        ks = [d for d in per.values() if key in d["name"]]
        if not ks:
            continue
        out["dram_bytes_per_launch"][name] = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ks) / len(ks)
        ms = [d["gpu__time_duration.sum"] / 1e6 for d in ks]
        out["ncu_ms_per_launch"][name] = sum(ms) / len(ms)
        out["share_of_pdgpu_kernels"][name] = sum(ms) / tot_ms
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
