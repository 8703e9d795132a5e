#!/usr/bin/env bash
# ORACLE / TEST INFRASTRUCTURE: regenerates tests/golden/* from the UNMODIFIED
# reference (oracle/_ref/ref_harness, built by `make -C oracle`). Run in the dev
# container (needs /root/reference); the outputs are committed.
set -euo pipefail
here=$(cd "$(dirname "$0")" && pwd)
root=$(cd "$here/.." && pwd)
make -s -C "$here" _ref/ref_harness
out="$root/tests/golden"
mkdir -p "$out"
h="$here/_ref/ref_harness"
"$h" digests > "$out/digests.json"
# name config n seed conc stream [chunk0 chunk1]
while read -r name cfg n seed conc stream c0 c1; do
  [[ -z "$name" || "$name" == \#* ]] && continue
  args=("$root/configs/$cfg" "$n" "$seed" "$conc" "$stream")
  [[ -n "${c0:-}" ]] && args+=("$c0" "$c1")
  "$h" trace "${args[@]}" | gzip -n -9 > "$out/trace_$name.txt.gz"
  echo "$name $cfg $n $seed $conc $stream ${c0:-} ${c1:-}"
done > "$out/traces.index" <<'LIST'
omni3_n100 omni3.json 100 7 16 1
omni3_full omni3.json 40 11 64 0
omni3_c64 omni3.json 100 7 64 1
omni3_tight omni3_tight.json 60 5 16 1
omni3_chunk1 omni3.json 30 3 16 1 1 1
thinker_only thinker_only.json 100 7 16 1
thinker_talker thinker_talker.json 100 7 16 1
ar_dit ar_dit.json 100 7 16 1
LIST
ls -la "$out"
