"""Per-source-line executed instructions and stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass` (one section per kernel)."""
import csv
import sys


def main(path, top=40, kernel_filter=""):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = fname = func = None
    out = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or (kernel_filter and kernel_filter not in (func or "")):
            continue
        try:
            samples, execd = int(r[4]), int(r[7])
        except (ValueError, IndexError):
            continue
        out.append((execd, samples, fname, r[0], r[1][:100]))
    ti = sum(x[0] for x in out) or 1
    ts = sum(x[1] for x in out) or 1
    print(f"total inst {ti}")
    for e, s, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{100 * e / ti:5.1f}% inst {100 * s / ts:5.1f}% samp  {f}:{ln:>4} | {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else "")
