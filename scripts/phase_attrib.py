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

SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'paper_1805_08995_b200', 'csrc', 'match_kernels.cuh')
MARKS = [  # (first line containing the text, phase of the lines from there on)
    ('void __launch_bounds__(kMatchThreads, 1) match_kernel', 'other'),
    ('for (;;) {', 'unit'),
    ('auto lookup_batch = ', 'lookup'),
    ('auto load_ids = ', 'ids'),
    ('uint32_t idn[LT];', 'loop'),
    ('} else if (tover <= 32u * kOverSlots) {', 'scan'),
    ('// ---- 3. ranking', 'rank'),
    ('// ---- long buckets', 'longbuckets'),
    ('if (!kMatch && emit) {', 'emit_dbg'),
    ('// ---- 4. verification', 'verify'),
    ('// batch boundary', 'loop'),
    ('st_raw = __reduce_add_sync', 'unit'),
]
_ranges = None
KERNEL_FIRST = KERNEL_LAST = 0


def _load_ranges():
    global _ranges, KERNEL_FIRST, KERNEL_LAST
    lines = open(SRC).read().splitlines()
    starts, at = [], 0
    for text, ph in MARKS:
        at = next(i for i in range(at, len(lines)) if text in lines[i])
        starts.append((at + 1, ph))
    end = next(i for i in range(at, len(lines)) if lines[i].startswith('}')) + 1
    KERNEL_FIRST, KERNEL_LAST = starts[0][0], end
    special = {}
    for i in range(starts[-2][0], starts[-1][0]):  # the loop tail calls the lookup and the id prefetch
        if 'lookup_batch(' in lines[i - 1]: special[i] = 'lookup'
        if 'load_ids(' in lines[i - 1]: special[i] = 'ids'
    for i in range(starts[4][0], starts[5][0]):    # ... and so does the loop head
        if 'lookup_batch(' in lines[i - 1]: special[i] = 'lookup'
        if 'load_ids(' in lines[i - 1]: special[i] = 'ids'
    _ranges = (starts, end, special)


def phase_of(line):
    if _ranges is None: _load_ranges()
    starts, end, special = _ranges
    if line is None or line < starts[0][0] or line > end: return 'other'
    if line in special: return special[line]
    ph = 'other'
    for first, name in starts:
        if line >= first: ph = name
    return ph


def main():
    src, lib, kernel, nq = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    _load_ranges()
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
            if f == 'match_kernels.cuh' and inl is None and KERNEL_FIRST <= l <= KERNEL_LAST:
                outer = l
        if outer is None:
            for f, l, inl in chain:
                if inl is not None and KERNEL_FIRST <= inl <= KERNEL_LAST: outer = inl
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
