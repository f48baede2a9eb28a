"""Executed-instruction mix per kernel from `ncu --page source --csv --print-source sass` output,
grouped by pipe class, normalised per unit (e.g. per butterfly)."""
import collections
import csv
import re
import sys

ALU = ('IADD3', 'LOP3', 'SEL', 'MOV', 'SHF', 'LEA', 'ISETP', 'PLOP3', 'P2R', 'R2P', 'PRMT', 'VIADD', 'IABS', 'IMNMX', 'FLO', 'BREV', 'POPC')
FMA_HEAVY = ('IMAD.WIDE', 'IMAD.HI')
FMA = ('IMAD', 'HFMA2', 'FFMA')


def classify(op):
    if op.startswith(FMA_HEAVY):
        return 'fma_heavy'
    if op.startswith(FMA):
        return 'fma'
    if op.startswith(('LDS', 'STS', 'LDG', 'STG', 'LD', 'ST', 'ATOM', 'RED')):
        return 'lsu'
    if op.startswith(ALU):
        return 'alu'
    if op.startswith('U'):
        return 'uniform'
    return 'other'


def main(path, units=None):
    rows = list(csv.reader(open(path)))
    kern = None
    data = collections.OrderedDict()
    hdr = None
    for row in rows:
        if row and row[0] == 'Kernel Name':
            kern = row[1]
            data[kern] = collections.Counter()
            hdr = None
            continue
        if row and row[0] == 'Address':
            hdr = row
            continue
        if hdr is None or not row:
            continue
        src = row[hdr.index('Source')]
        n = int(row[hdr.index('Thread Instructions Executed')] or 0)
        m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', src)
        if m:
            data[kern][m.group(2)] += n
    for k, c in data.items():
        tot = sum(c.values())
        cls = collections.Counter()
        for op, v in c.items():
            cls[classify(op)] += v
        print('===', k[:80], 'thread-instr', tot)
        u = units or 1
        print('   per unit: total %.1f | ' % (tot / u) + ', '.join('%s %.1f' % (a, b / u) for a, b in cls.most_common()))
        print('   top:', ', '.join('%s %.1f' % (a, b / u) for a, b in c.most_common(22)))


if __name__ == '__main__':
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
