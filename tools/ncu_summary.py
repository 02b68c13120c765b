"""Key metrics from an ncu details CSV (tools/prof2.sh output)."""
import csv
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Achieved Occupancy', 'Registers Per Thread',
        'Grid Size', 'Block Size', 'Compute (SM) Throughput', 'L2 Hit Rate', 'Theoretical Occupancy',
        'Dynamic Shared Memory Per Block', 'Warp Cycles Per Issued Instruction', 'Issue Slots Busy',
        'Waves Per SM', 'Executed Ipc Active']
for f in sys.argv[1:]:
    print("==", f)
    for r in csv.reader(open(f)):
        if len(r) > 14 and r[12] in WANT:
            print(f"  {r[12]:40s} {r[14]:>12s} {r[13]}")
