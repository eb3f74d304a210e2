"""Per-source-line stall samples / instruction counts from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep [kernel-substring] [--top N]
Extracts the cubin from libfmap_cuda.so, maps SASS offsets to lines with
`nvdisasm -g`, and joins them with ncu's SASS source page.
"""
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    rep = sys.argv[1]
    ksub = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "chol_solve_kernelILi0"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_2604_10377_b200/libfmap_cuda.so")],
                   cwd=tmp, capture_output=True)
    lines = {}
    for cub in tmp.glob("*.cubin"):
        txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout
        inside, cur = False, None
        for ln in txt.splitlines():
            if ln.startswith(".text."):
                inside = ksub in ln
                continue
            if not inside:
                continue
            m = re.search(r'## File "(.*)", line (\d+)', ln)
            if m:
                cur = (Path(m.group(1)).name, int(m.group(2)))
                continue
            mo = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
            if mo and cur:
                lines[int(mo.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {x: i for i, x in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h)]
    base = int(data[0][ix["Address"]], 16)
    agg = {}
    for r in data:
        key = lines.get(int(r[ix["Address"]], 16) - base, ("?", 0))
        a = agg.setdefault(key, [0, 0])
        a[0] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        a[1] += int(r[ix["Instructions Executed"]] or 0)
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    srcs = {}
    print(f"{'file:line':28s} stall%  instr%")
    for (f, ln), (s, n) in sorted(agg.items(), key=lambda x: -(x[1][0] / ts + x[1][1] / ti))[:top]:
        p = ROOT / "paper_2604_10377_b200/csrc" / f
        if f not in srcs and p.exists():
            srcs[f] = p.read_text().split("\n")
        text = srcs.get(f, [""] * (ln + 1))[ln - 1].strip() if ln else ""
        print(f"{f + ':' + str(ln):28s} {100*s/ts:5.1f}  {100*n/ti:5.1f}  {text[:80]}")


if __name__ == "__main__":
    main()
