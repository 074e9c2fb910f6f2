"""Attribute ncu warp-stall samples (`--page source --csv --print-source sass`) to source lines.

The report's SASS page carries per-instruction samples but no line numbers; the line info comes from
`nvdisasm -g` of the same build's cubin (compiled with -lineinfo).  Usage:
  python scripts/sass_lines.py <sass.csv> <nvdisasm -g output> <kernel-name substring> [top]
Prints the source lines with the most samples: total, not-issued, the three largest stall reasons,
and the executed warp instructions."""
import collections
import csv
import re
import sys


def kernel_blocks(path):
    """Yield (kernel name, header, rows) per kernel section of the ncu source CSV."""
    name, hdr, rows = None, None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            if name is not None:
                yield name, hdr, rows
            name, hdr, rows = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif r:
            rows.append(r)
    if name is not None:
        yield name, hdr, rows


def line_map(disasm, mangled_sub):
    """offset -> 'file:line' for the function whose mangled name contains mangled_sub."""
    m, cur, inside = {}, "?", False
    for ln in open(disasm):
        if ln.startswith("//----") and ".text." in ln:
            inside = mangled_sub in ln
            continue
        if not inside:
            continue
        g = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = f"{g.group(1).split('/')[-1]}:{g.group(2)}"
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    csvp, dis, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    mangled = sys.argv[5] if len(sys.argv) > 5 else None
    for name, hdr, rows in kernel_blocks(csvp):
        if kname not in name:
            continue
        ix = {h: i for i, h in enumerate(hdr)}
        base = int(rows[0][0], 16)
        lm = line_map(dis, mangled or kname)
        tot = collections.Counter()
        nis = collections.Counter()
        ins = collections.Counter()
        st = collections.defaultdict(collections.Counter)
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        for r in rows:
            off = int(r[0], 16) - base
            key = lm.get(off, "?")
            tot[key] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            nis[key] += int(r[ix["Warp Stall Sampling (Not-issued Samples)"]] or 0)
            ins[key] += int(r[ix["Instructions Executed"]] or 0)
            for h in stall_cols:
                v = int(r[ix[h]] or 0)
                if v:
                    st[key][h[6:]] += v
        T = sum(tot.values())
        print(f"== {name}: {T} samples, {sum(ins.values())} warp instructions")
        for key, v in tot.most_common(top):
            reasons = ", ".join(f"{k} {c}" for k, c in st[key].most_common(3))
            print(f"{100.0 * v / max(T, 1):5.1f}%  {key:28s} samples {v:6d} not-issued {nis[key]:6d} inst {ins[key]:9d}  [{reasons}]")
        break


if __name__ == "__main__":
    main()
