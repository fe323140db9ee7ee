"""Top SASS instructions by warp-stall samples from an ncu report (--page source)."""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(out.splitlines()))
    hdr = None
    res = []
    for i, r in enumerate(rd):
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except ValueError:
                continue
            res.append((samp, i, r[1][:90]))
    tot = sum(s for s, _, _ in res) or 1
    for s, i, src in sorted(res, reverse=True)[:top]:
        print(f"{s / tot * 100:5.1f}%  #{i:5d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
