"""Summarise an .ncu-rep: key metrics per profiled kernel launch."""
import csv, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2].split(',') if len(sys.argv) > 2 else [
    'Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate',
    'L2 Hit Rate', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
    'Issue Slots Busy', 'Warp Cycles Per Issued Instruction', 'L1/TEX Cache Throughput',
    'L2 Cache Throughput', 'Executed Ipc Active']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, idi, mi, ui, vi = (h.index(x) for x in ('Kernel Name', 'ID', 'Metric Name', 'Metric Unit', 'Metric Value'))
seen = set()
for row in r[1:]:
    if row[mi] in want and (row[idi], row[mi]) not in seen:
        seen.add((row[idi], row[mi]))
        print(f"{row[idi]:>3} {row[ki].split('(')[0][:28]:28s} {row[mi]:36s} {row[vi]:>14s} {row[ui]}")
