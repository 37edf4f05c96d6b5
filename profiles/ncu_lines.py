"""Per-CUDA-source-line hot spots from an ncu report (cuda,sass source view):
warp-stall samples, shared-memory excess wavefronts and instruction counts.
usage: python profiles/ncu_lines.py report.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys


def main(rep, kern, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, lines = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif len(r) > 2 and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r[2:])}
        elif hdr and len(r) > 4 and r[0] not in ("", "Function Name"):
            def num(k):
                try:
                    return float(r[2 + hdr[k]])
                except (ValueError, KeyError, IndexError):
                    return 0.0
            stalls = sorted(((num(k), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k),
                            reverse=True)[:3]
            lines.append((fname, r[0], r[1].strip()[:60], num("Warp Stall Sampling (All Samples)"),
                          num("L1 Wavefronts Shared Excessive"), num("Instructions Executed"),
                          " ".join(f"{n}:{v:.0f}" for v, n in stalls if v > 0)))
    tot = sum(x[3] for x in lines) or 1
    print(f"total stall samples {tot:.0f}")
    for f, ln, src, s, ex, ins, st in sorted(lines, key=lambda x: -x[3])[:n]:
        print(f"{f}:{ln:>5} {100 * s / tot:5.1f}% exc_sh={ex:>9.0f} inst={ins:>10.0f} [{st}]  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
