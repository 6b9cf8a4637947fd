"""Aggregate warp-stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    fname = None
    out = []
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            samples = int(r[4])
            execd = int(r[7])
        except (ValueError, IndexError):
            continue
        out.append((samples, fname, r[0], execd, r[1][:110]))
    tot = sum(x[0] for x in out) or 1
    for s, f, ln, ex, src in sorted(out, reverse=True)[:top]:
        print(f"{100*s/tot:5.1f}% {f}:{ln:>4} inst={ex:>11} | {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
