"""Per-source-line instruction counts and stall samples of one kernel: joins the SASS page of an
ncu report (instruction order) with nvdisasm's line table of the same kernel in the built object.

    python profiles/source_lines.py gpurun_out/x.ncu-rep paper_2406_04210_b200/lib/obj/nlist.o \
        k_list_cells_ballotILi8ELb1 [top]

Runs in the build container (no GPU): needs ncu, cuobjdump and nvdisasm on PATH."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[head]
    ia, ii, isamp = h.index("Address"), h.index("Instructions Executed"), h.index("# Samples")
    res = []
    for r in rows[head + 1:]:
        if len(r) <= max(ii, isamp) or not r[ia].startswith("0x"):
            continue
        res.append((int(r[ia], 16), int(r[ii] or 0), int(r[isamp] or 0), r[h.index("Source")]))
    base = res[0][0]
    return [(a - base, n, s, txt) for a, n, s, txt in res]


def line_table(obj, pattern):
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp,
                       capture_output=True)
        cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
        text = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)],
                              capture_output=True, text=True).stdout
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and pattern in l)
    table, cur = {}, None
    for l in lines[start + 1:]:
        if l.startswith("//---------------------"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:
            # inlined code: keep the innermost location (the last one printed)
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
        if m:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    rep, obj, pattern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = sass_rows(rep)
    table = line_table(obj, pattern)
    per_line = {}
    total_n = total_s = 0
    for off, n, s, _ in rows:
        loc = table.get(off, ("?", 0))
        a = per_line.setdefault(loc, [0, 0])
        a[0] += n
        a[1] += s
        total_n += n
        total_s += s
    src_cache = {}
    print(f"total warp instructions {total_n}, stall samples {total_s}")
    for loc, (n, s) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        fname, line = loc
        text = ""
        path = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "..", "csrc", fname)
        if os.path.exists(path):
            src_cache.setdefault(path, open(path).read().splitlines())
            if 0 < line <= len(src_cache[path]):
                text = src_cache[path][line - 1].strip()[:90]
        print(f"{100 * n / total_n:5.1f} % instr {100 * s / max(total_s, 1):5.1f} % samples  "
              f"{fname}:{line:<5} {text}")


if __name__ == "__main__":
    main()
