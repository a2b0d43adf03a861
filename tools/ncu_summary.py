"""Print the key ncu --set full metrics of a report (run here, on CPU)."""
import csv
import subprocess
import sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Occupancy', 'Memory Workload Analysis', 'Scheduler Statistics',
            'Warp State Statistics', 'Compute Workload Analysis', 'Launch Statistics')
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'launch__registers_per_thread',
       'launch__grid_size', 'launch__block_size', 'sm__warps_active.avg.pct_of_peak_sustained_active',
       'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active']


def main(rep, full=False):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get('Section Name') in SECTIONS and (full or d['Section Name'] != 'Launch Statistics'):
            print(f"{d['Section Name'][:22]:22s} | {d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}")
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    for k, u, x in zip(h, units, v):
        if k in RAW or k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
            if k.startswith('smsp__pcsamp') and float(x or 0) < 1:
                continue
            print(f"raw | {k} = {x} {u}")


if __name__ == '__main__':
    main(sys.argv[1], '--full' in sys.argv)
