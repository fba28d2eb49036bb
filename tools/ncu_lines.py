"""Per-source-line executed instructions and stall samples of one kernel in an
ncu report (the cuda,sass source page), optionally diffed against a second report
by source text:  python tools/ncu_lines.py A.ncu-rep [B.ncu-rep] [--top N]"""
import csv
import io
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, hdr = {}, None
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr and r and r[0] not in ("", "File Path", "Function Name") and len(r) > ie:
            key = r[1].strip()
            try:
                a, b = int(r[ie]), int(r[sm])
            except ValueError:
                continue
            x = res.setdefault(key, [0, 0, r[0]])
            x[0] += a
            x[1] += b
    return res


def main():
    argv = sys.argv[1:]
    if "--top" in argv:
        k = argv.index("--top")
        argv = argv[:k] + argv[k + 2:]
    args = [a for a in argv if not a.startswith("--")]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    A = lines(args[0])
    if len(args) == 1:
        tot = sum(v[0] for v in A.values()); ts = sum(v[1] for v in A.values())
        for k, v in sorted(A.items(), key=lambda kv: -kv[1][0])[:top]:
            print(f"{v[0]:>12d} {100*v[0]/tot:5.1f}% samp {100*v[1]/max(ts,1):5.1f}%  L{v[2]:>4} {k[:100]}")
        return
    B = lines(args[1])
    keys = set(A) | set(B)
    d = sorted(keys, key=lambda k: -abs(A.get(k, [0])[0] - B.get(k, [0])[0]))
    print("total", sum(v[0] for v in A.values()), sum(v[0] for v in B.values()))
    for k in d[:top]:
        a, b = A.get(k, [0, 0, "-"]), B.get(k, [0, 0, "-"])
        print(f"{a[0]:>12d} {b[0]:>12d} {b[0]-a[0]:>+11d}  {k[:100]}")


if __name__ == "__main__":
    main()
