# per-launch device times of one workload's step (ncu launch list), default lib and OPCFE_LIB variants
cd $GRAFT_REPO_ROOT
W=${1:-C2}; FR=${2:-8}
for L in "" dev/ab/*.so; do
  tag=$(basename "${L:-default}" .so)
  env ${L:+OPCFE_LIB=$PWD/$L} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_${W}_$tag.csv python bench.py --workload $W --frames $FR --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python - "$W" "$tag" <<'PY'
import csv, sys, collections
W, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(f"gpurun_out/ll_{W}_{tag}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
tail = seq[-len(seq) // 5:]
agg = collections.OrderedDict()
for k, v in tail:
    n = k.split("(")[0][-40:]
    agg.setdefault(n, []).append(v)
print(tag, {k: (len(v), round(sum(v) / len(v) / 1000, 2)) for k, v in agg.items()})
PY
done
