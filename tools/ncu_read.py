"""Summarise an ncu report: key speed-of-light / occupancy metrics per kernel launch."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy', 'Registers Per Thread',
        'L2 Hit Rate', 'Issue Slots Busy', 'Grid Size', 'Theoretical Occupancy', 'L1/TEX Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Memory Throughput']


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, idi, mn, mv, mu = (hdr.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    cur = None
    for row in rows[1:]:
        if row[mn] in WANT:
            k = (row[idi], row[ki][:60])
            if k != cur:
                print("==", *k)
                cur = k
            print("   ", row[mn], row[mv], row[mu])


if __name__ == "__main__":
    main(sys.argv[1])
