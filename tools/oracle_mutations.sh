#!/bin/bash
# Mutation check of the oracle pins: apply one plausible mistake at a time to
# a scratch copy of oracle/oracle.c and confirm that `pytest -m "not gpu"`
# fails.  Usage: tools/oracle_mutations.sh   (CPU only, ~1 min)
set -u
REPO=$(cd "$(dirname "$0")/.." && pwd)
SCR=$(mktemp -d)
run() {
  rm -rf "$SCR/r" && cp -r "$REPO" "$SCR/r" && rm -f "$SCR/r/oracle/liboracle.so"
  sed -i "$1" "$SCR/r/oracle/oracle.c"
  if cmp -s "$SCR/r/oracle/oracle.c" "$REPO/oracle/oracle.c"; then echo "$2: pattern did not apply"; return; fi
  res=$(cd "$SCR/r" && timeout 600 python -m pytest tests -q -m "not gpu" -k "oracle_pins" 2>&1 | tail -1)
  echo "$2: $res"
}
run 's/4.5 \* cu \* cu/4.0 * cu * cu/' "equilibrium 4.5 -> 4.0"
run 's/- 1.5 \* usq/- 1.0 * usq/' "equilibrium 1.5 -> 1.0"
run 's/1.0 + 3.0 \* cu/1.0 - 3.0 * cu/' "equilibrium sign of 3 c.u"
run 's/v = v + 6.0 \* W\[i\]/v = v - 6.0 * W[i]/' "lid term sign"
run 's/if (sz >= nz) {/if (sz < 0) {/' "lid on the wrong z face"
run 's/int sx = gx - C\[i\]\[0\]/int sx = gx + C[i][0]/' "push instead of pull in x"
run 's/v = fstar\[idx(OPP\[i\], x, y, z/v = fstar[idx(i, x, y, z/' "bounce-back without opp"
run 's/1.0 \/ tau,/1.0 \/ (tau + 0.0001),/' "tau convention"
run 's/{-1, 0, -1}, {-1, 0, 1}/{-1, 0, 1}, {-1, 0, -1}/' "directions 6,7 transposed"
run 's/feq\[0\] = rest;/feq[0] = W[0] * rho * (1.0 - 1.5 * usq);/' "no rest-population closure"
run 's/u\[a\] = j\[a\] \/ r;/u[a] = j[a] \/ (r + 1e-9);/' "perturbed velocity division"
run 's/a = b;$/a = a;/' "run: lattices not swapped"
run 's/if (a != f) memcpy/if (0) memcpy/' "run: odd-step result not copied back"
rm -rf "$SCR"
