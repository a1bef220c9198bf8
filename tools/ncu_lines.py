"""Per-CUDA-source-line stall samples from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys


def lines(rep, top=40):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout.splitlines()
    res = []
    cur_file = None
    hdr = None
    for row in csv.reader(out):
        if not row:
            continue
        if row[0] == 'File Path':
            cur_file = row[1].split('/')[-1]
            continue
        if row[0] == 'Line No':
            hdr = row
            continue
        if hdr is None or row[0] == '' or row[0] == 'Function Name':
            continue
        try:
            s = float(row[4])
        except (ValueError, IndexError):
            continue
        res.append((s, cur_file, row[0], row[1].strip()[:90]))
    tot = sum(r[0] for r in res) or 1
    res.sort(reverse=True)
    for s, f, ln, src in res[:top]:
        print(f"{100*s/tot:5.1f}%  {f}:{ln:5s} {src}")


if __name__ == '__main__':
    lines(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
