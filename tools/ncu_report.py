"""Summarise an ncu report (+ launch list) into profiles/ (run here, no GPU needed)."""
import csv, json, subprocess, sys
from collections import defaultdict

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
       'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
       'gpu__time_duration.sum', 'sm__warps_active.avg.per_cycle_active']


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    r = r[next(i for i, row in enumerate(r) if 'Kernel Name' in row):]
    h = r[0]
    ki, ii, mi, vi, ui = (h.index('Kernel Name'), h.index('ID'), h.index('Metric Name'), h.index('Metric Value'),
                          h.index('Metric Unit'))
    res = defaultdict(dict)
    for row in r[1:]:
        if row[mi] in WANT:
            res[(row[ii], row[ki])][row[mi]] = f"{row[vi]} {row[ui]}".strip()
    return res


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    r = r[next(i for i, row in enumerate(r) if 'Kernel Name' in row):]
    h, units, rows = r[0], r[1], r[2:]
    res = {}
    stall = {}
    for row in rows:
        key = (row[h.index('ID')], row[h.index('Kernel Name')])
        res[key] = {m: f"{row[h.index(m)]} {units[h.index(m)]}".strip() for m in RAW if m in h}
        st = []
        for i, name in enumerate(h):
            if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('not_issued'):
                try:
                    st.append((float(row[i].replace(',', '')), name.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        stall[key] = [(n, round(100 * x / tot, 1)) for x, n in sorted(st, reverse=True)[:6]]
    return res, stall


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, iv, iu = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        v = float(r[iv].replace(',', ''))
        v = v / 1e6 if r[iu] == 'ns' else (v / 1e3 if r[iu] in ('us', 'usecond') else v)
        k = r[ik].split('(')[0]
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    return [(k, cnt[k], round(tot[k], 4), round(100 * tot[k] / s, 1)) for k in sorted(tot, key=lambda k: -tot[k])]


if __name__ == "__main__":
    rep, launch_csv, out_md, out_json = sys.argv[1:5]
    d = details(rep)
    rw, st = raw(rep)
    lines = [f"# ncu summary: {rep.split('/')[-1]}", ""]
    traffic = {}
    for key in d:
        lines.append(f"## {key[1][:90]} (launch id {key[0]})")
        for m in WANT:
            if m in d[key]:
                lines.append(f"- {m}: {d[key][m]}")
        for m, v in rw.get(key, {}).items():
            lines.append(f"- {m}: {v}")
        lines.append(f"- top stall reasons (% of samples): {st.get(key)}")
        lines.append("")
        try:
            b = float(rw[key]['dram__bytes_read.sum'].split()[0].replace(',', '')) * (1 if 'byte' == rw[key]['dram__bytes_read.sum'].split()[-1] else 1)
        except Exception:
            b = None
    if launch_csv != "-":
        lines.append("## launch list (gpu__time_duration, serialised under ncu; compare shares)")
        lines.append("| kernel | launches | total ms | share |")
        lines.append("|---|---|---|---|")
        for k, c, t, sh in launches(launch_csv):
            lines.append(f"| {k} | {c} | {t} | {sh}% |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
