# A/B of gather/scatter library variants on C5cycle: bash scripts/ab_combi.sh name1 name2 ...
# (name = lib_var/<name>.so, "cur" = lib/libsgh.so)
for v in "$@"; do
  if [ $v = cur ]; then unset SGH_LIB_PATH; else export SGH_LIB_PATH=$PWD/lib_var/$v.so; fi
  timeout 300 python bench.py --workload C5cycle --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.json 2>/tmp/x.err
  python - $v <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
ks=d["kernels"]
print(sys.argv[1], round(d["ms_per_step"],1), {k: round(ks[k]["share_of_step"]*d["ms_per_step"],2) for k in ("gather","scatter")})
PY
done
