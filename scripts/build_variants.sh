#!/bin/bash
# Build tuning variants of libsgh in parallel: each arg is "name DEF=V DEF2=V2 ..."
# -> paper_1309_0392_b200/lib/var_<name>.so  (select one with SGH_LIB_PATH)
root=$(cd "$(dirname "$0")/.." && pwd)
pids=()
for v in "$@"; do
  set -- $v; name=$1; shift; defs=""
  for d in "$@"; do defs="$defs -D $d"; done
  python $root/paper_1309_0392_b200/build.py --out $root/paper_1309_0392_b200/lib/var_$name.so $defs > /tmp/bvar_$name.log 2>&1 &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
exit $rc
