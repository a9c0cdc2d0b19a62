# Round 2 ncu pass: launch list of the default bench command, and one
# --set full capture per bench kernel (headline, C3 routes, C2, bits).
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c4.csv python bench.py > gpurun_out/r2_17_bench_under_ncu.json 2> gpurun_out/r2_17_bench_under_ncu.err
for spec in "unit_f32 32" "bits 32" "gauss_f32 30" "logn_f32 30" "gauss_f32_precise 30" "gauss_f32_exact 30" "mrg_f64 28"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_kernel|philox_kernel" -c 1 -s 1 -o gpurun_out/r2_ncu_$1_2p$2 python tools/ncu_target.py $1 $2 3 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/r2_ncu_$1_2p$2.ncu-rep > gpurun_out/r2_ncu_$1_2p$2.txt 2>&1
done
ls -la gpurun_out/*.ncu-rep
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r2_launches_bench_c4.csv")))
hdr = None
from collections import defaultdict
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows:
    if "Kernel Name" in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][:80]
            tot[k] += float(d["Metric Value"].replace(",", "")); cnt[k] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"{v/T:6.3f} share  {cnt[k]:6d} launches  {v/cnt[k]/1e3:10.1f} us avg  {k}")
PY
for f in gpurun_out/r2_ncu_*.txt; do echo "== $f"; head -22 $f; done
