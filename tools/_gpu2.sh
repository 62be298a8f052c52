cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 --cpu-seconds 3 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
tail -3 gpurun_out/g2_bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/g2_bench.json"))
print("value", round(d["value"]), "frac", round(d["roofline"]["frac"], 3), "e2e", d["e2e"]["value"], d.get("shard_checksums"))
print(d["cpu_baseline"])
for s in d.get("suite", []):
    print(f'{s["workload"]:22s} {s["elements_per_s"]:12.0f} el/s  roof {s["roofline_frac"]:.3f}')
PY
for v in 0 1; do
  HXG_V3_P7=$v python bench.py --workload c5_h1_p7_general --elements 4096 --no-suite --no-cpu --e2e-steps -1 --steps 5 > gpurun_out/g2_h1p7_v3$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/g2_h1p7_v3$v.json'));print('H1p7 v3=$v', d['value'], d['roofline']['frac'])"
done
