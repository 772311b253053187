import csv, json, sys
for f in ['gpurun_out/exp_bench_c3.json', 'gpurun_out/exp_bench_C2.json', 'gpurun_out/exp_bench_C4.json']:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'unreadable', e); continue
    r = d['roofline']
    print(f, 'step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['ms_per_step'], 3), 'root',
          round(r['mean_launch_ms'], 3), 'frac', round(r['frac'], 4), d['clocks']['sm_mhz'], d['clocks']['reasons'])
def load(f):
    rows = list(csv.reader(open(f)))
    return dict(zip(rows[0], rows[-1]))
a = load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/c3_wtile_raw.csv')
b = load('gpurun_out/c3_exp_raw.csv')
keys = [k for k in a if ('issue_stalled' in k and 'per_issue_active' in k) or k in (
    'gpu__time_duration.sum', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
    'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
    'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
    'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread')]
for k in keys:
    if a.get(k) not in ('0', None) or b.get(k) not in ('0', None):
        print(k.replace('smsp__average_warps_issue_stalled_', ''), a.get(k), b.get(k))
