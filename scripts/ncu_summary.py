"""Summarise an .ncu-rep (raw page) into the metrics we track; optional source hot spots."""
import csv, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'launch__shared_mem_per_block_dynamic', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__pcsamp_warps_issue_stalled_long_scoreboard', 'smsp__pcsamp_warps_issue_stalled_short_scoreboard',
        'smsp__pcsamp_warps_issue_stalled_wait', 'smsp__pcsamp_warps_issue_stalled_selected',
        'smsp__pcsamp_warps_issue_stalled_not_selected', 'smsp__pcsamp_warps_issue_stalled_math_pipe_throttle',
        'smsp__pcsamp_warps_issue_stalled_lg_throttle', 'smsp__pcsamp_warps_issue_stalled_mio_throttle',
        'smsp__pcsamp_warps_issue_stalled_branch_resolving', 'smsp__pcsamp_warps_issue_stalled_barrier',
        'smsp__pcsamp_warps_issue_stalled_dispatch_stall', 'smsp__pcsamp_warps_issue_stalled_no_instructions',
        'smsp__pcsamp_warps_issue_stalled_drain', 'smsp__pcsamp_warps_issue_stalled_tex_throttle']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({n: (v[i], units[i]) for i, n in enumerate(h) if i < len(v)})
    return res


def hot(rep, n=25):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]; data = [r for r in rows[2:] if len(r) == len(h)]
    iw, isrc = h.index('Warp Stall Sampling (All Samples)'), h.index('Source')
    tot = sum(float(r[iw] or 0) for r in data) or 1
    for k, r in sorted(enumerate(data), key=lambda kr: -float(kr[1][iw] or 0))[:n]:
        prev = data[k - 1][isrc] if k else ''
        print(f"  {float(r[iw]) / tot * 100:5.1f}%  {r[isrc][:58]:58s} | prev {prev[:40]}")


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        if rep == '--hot':
            continue
        for k in raw(rep):
            print('==', rep, k.get('Kernel Name', ('?',))[0][:80])
            for w in WANT:
                if w in k:
                    print(f"  {w:66s} {k[w][0]} {k[w][1]}")
        if '--hot' in sys.argv:
            hot(rep)
