"""Top warp-stall SASS lines of one kernel launch in an ncu report.

python tools/ncu_stalls.py REPORT.ncu-rep KERNEL_REGEX [LAUNCH_SKIP] [TOP]
(-lineinfo builds; --page source --print-source sass)
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kern}", "--launch-skip", skip,
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[hi]
    isrc, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        if not r or not r[0].startswith("0x"):
            break  # first copy only
        data.append((r[isrc].strip(), int(r[ie] or 0), int(r[iss] or 0)))
    tot = sum(d[2] for d in data)
    print(f"{len(data)} SASS lines, {tot} stall samples, {sum(d[1] for d in data)} warp instructions")
    for i in sorted(sorted(range(len(data)), key=lambda i: -data[i][2])[:top]):
        s, e, smp = data[i]
        print(f"{i:5d} {smp:6d} {100.0 * smp / max(tot, 1):5.1f}% {e:10d}  {s[:90]}")


if __name__ == "__main__":
    main()
