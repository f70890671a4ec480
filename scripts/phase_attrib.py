#!/usr/bin/env python
"""Per-phase attribution of the match kernel's executed warp instructions.

Joins the per-SASS-instruction "Instructions Executed" column of an ncu source page
(ncu -i X.ncu-rep --page source --csv) with the line table of the cubin (nvdisasm -gi -c),
takes the OUTERMOST line of every instruction's inline chain (the line of match_kernel's body that
the instruction belongs to) and sums by phase.

Usage: python scripts/phase_attrib.py SOURCE.csv LIB_OR_CUBIN KERNEL_MANGLED_SUBSTR QUERIES_PER_LAUNCH [out.json]
"""
import csv, json, re, subprocess, sys, tempfile, os, collections

def sass_lines(lib, kernel):
    tmp = tempfile.mkdtemp()
    if lib.endswith('.so'):
        subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(lib)], cwd=tmp, check=True, stdout=subprocess.DEVNULL)
        cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith('.cubin')]
    else:
        cubins = [lib]
    for cb in cubins:
        txt = subprocess.run(['nvdisasm', '-gi', '-c', cb], capture_output=True, text=True).stdout
        key = '.text.' + kernel
        if key + ':' not in txt and key not in txt:
            continue
        out, on, chain = {}, False, []
        pending = []
        for ln in txt.splitlines():
            if ln.startswith('.text.'):
                on = kernel in ln
                continue
            if ln.startswith('//-----') and on and kernel not in ln:
                on = False
            if not on:
                continue
            m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
            if m:
                pending.append((os.path.basename(m.group(1)), int(m.group(2)), m.group(4) and int(m.group(4))))
                continue
            m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
            if m:
                if pending:
                    chain = pending
                    pending = []
                addr = int(m.group(1), 16)
                out[addr] = (chain, m.group(2).strip())
        if out:
            return out
    raise SystemExit('kernel not found in ' + lib)

def phase_of(line):
    if line is None: return 'other'
    if 443 <= line <= 491: return 'lookup'
    if 494 <= line <= 500: return 'ids'
    if 395 <= line <= 433 or 435 <= line <= 438: return 'unit'
    if line in (505, 703): return 'lookup'
    if line in (506, 704, 519): return 'ids'
    if 502 <= line <= 529 or 700 <= line <= 706: return 'loop'
    if 531 <= line <= 566: return 'scan'
    if 568 <= line <= 610: return 'rank'
    if 611 <= line <= 679: return 'longbuckets'
    if 681 <= line <= 690: return 'emit_dbg'
    if 693 <= line <= 698: return 'verify'
    if 709 <= line <= 717: return 'unit'
    return 'other'

def main():
    src, lib, kernel, nq = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    table = sass_lines(lib, kernel)
    rows = list(csv.reader(open(src)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == 'Address')
    hdr = rows[hdr_i]
    ci, cs = hdr.index('Instructions Executed'), hdr.index('Source')
    cw = hdr.index('L1 Wavefronts Shared') if 'L1 Wavefronts Shared' in hdr else None
    base = None
    per_phase = collections.Counter(); per_line = collections.Counter(); per_op = collections.defaultdict(collections.Counter)
    total = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= ci or not r[ci]: continue
        addr = int(r[0], 16) if r[0].startswith('0x') else int(r[0])
        if base is None: base = addr
        n = int(float(r[ci]))
        off = addr - base
        chain, text = table.get(off, ([], r[cs]))
        # outermost line in match_kernels.cuh inside the kernel body (>= 365); else innermost known
        outer = None
        for f, l, inl in chain:
            if f == 'match_kernels.cuh' and inl is None and l >= 365 and l <= 718:
                outer = l
        if outer is None:
            for f, l, inl in chain:
                if inl is not None and 365 <= inl <= 718: outer = inl
        ph = phase_of(outer)
        op = text.split()[0] if not text.startswith('@') else text.split()[1]
        op = op.split('.')[0]
        per_phase[ph] += n; per_line[outer] += n; per_op[ph][op] += n
        total += n
    res = {'queries_per_launch': nq, 'warp_instructions_per_query': total / nq,
           'phases': {p: round(c / nq, 2) for p, c in per_phase.most_common()},
           'top_ops_per_phase': {p: {o: round(c / nq, 2) for o, c in per_op[p].most_common(12)} for p in per_phase},
           'lines': {str(l): round(c / nq, 2) for l, c in sorted(per_line.items(), key=lambda kv: -kv[1])[:60]}}
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 5:
        json.dump(res, open(sys.argv[5], 'w'), indent=1)

if __name__ == '__main__':
    main()
