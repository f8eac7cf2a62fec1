"""Hot spots of an ncu report (needs -lineinfo + --import-source on): CUDA
source lines (or SASS with --sass) ranked by warp-stall samples, with the
dominant stall reasons.

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [--sass] [--top 30] [--kernel N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    sass = "--sass" in sys.argv
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
    if "--kernel" in sys.argv:
        cmd += ["--print-kernel-base", "function", "-k", sys.argv[sys.argv.index("--kernel") + 1]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, fname, items = None, "?", []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if "Warp Stall Sampling (All Samples)" in r:
            h = r
            si = r.index("Warp Stall Sampling (All Samples)")
            stalls = [i for i, c in enumerate(r) if c.startswith("stall_") and "Not Issued" not in c]
            continue
        if h is None or len(r) <= si:
            continue
        is_line = r[0] != ""
        if is_line == sass:
            continue
        try:
            s = float(r[si])
        except ValueError:
            continue
        label = f"{fname}:{r[0]}" if is_line else r[2][-6:]
        text = r[1] if is_line else r[3]
        reasons = sorted(((float(r[i] or 0) if r[i] not in ("", "-") else 0.0, h[i][6:])
                          for i in stalls), reverse=True)[:3]
        items.append((s, label, text.strip(), reasons))
    tot = sum(x[0] for x in items)
    print(f"total samples {tot:.0f}")
    for s, label, text, reasons in sorted(items, key=lambda x: -x[0])[:top]:
        rs = " ".join(f"{n}={v / max(s, 1):.0%}" for v, n in reasons if v > 0)
        print(f"{s / max(tot, 1):6.1%} {label:>22} {text[:80]:80s} {rs}")


if __name__ == "__main__":
    main()
