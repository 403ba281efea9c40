"""Summaries of ncu outputs for profiles/ (run in the build container)."""
import collections, csv, subprocess, sys

def launches(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, mv, mu = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mv: continue
        try: v = float(r[mv].replace(',', ''))
        except ValueError: continue
        scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3,
                 's': 1e6, 'second': 1e6}[r[mu]]
        name = r[ki].split('(')[0].replace('void ', '')
        tot[name] += v * scale; cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append("| `%s` | %d | %.1f | %.1f%% | %.2f |" % (k[:70], cnt[k], v, 100 * v / T, v / cnt[k]))
    out.append("| **total** | %d | %.1f | 100%% | |" % (sum(cnt.values()), T))
    return "\n".join(out)

def full(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size',
            'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'lts__t_bytes.sum']
    idx = [h.index(w) for w in want if w in h]
    out = ["| " + " | ".join(h[i] for i in idx) + " |", "|" + "---|" * len(idx),
           "| " + " | ".join(rows[1][i] for i in idx) + " |"]
    for r in rows[2:]:
        out.append("| " + " | ".join(r[i].split('(')[0][:48] for i in idx) + " |")
    return "\n".join(out)

if __name__ == '__main__':
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == 'launches' else full(path))
