#!/bin/bash
# Mutation check of the oracle pins: apply one plausible mistake at a time to
# a scratch copy of oracle/oracle.c and confirm that `pytest -m "not gpu"`
# fails.  Usage: tools/oracle_mutations.sh   (CPU only, ~1 min)
set -u
REPO=$(cd "$(dirname "$0")/.." && pwd)
SCR=$(mktemp -d)
run() {  # run <sed expression> <label> [file under oracle/, default oracle.c]
  local f=${3:-oracle.c}
  rm -rf "$SCR/r" && cp -r "$REPO" "$SCR/r" && rm -f "$SCR/r/oracle/liboracle.so"
  sed -i "$1" "$SCR/r/oracle/$f"
  if cmp -s "$SCR/r/oracle/$f" "$REPO/oracle/$f"; then echo "$2: pattern did not apply"; return; fi
  res=$(cd "$SCR/r" && timeout 600 python -m pytest tests -q -m "not gpu" -k "oracle_pins or oracle_dqq" 2>&1 | tail -1)
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
# the other-lattice oracle (oracle_dqq.c)
run 's|wc = 1.0 / 72.0;|wc = 1.0 / 64.0;|' "D3Q15 corner weight" oracle_dqq.c
run 's|wf = 1.0 / 54.0; wc = 1.0 / 216.0;|wf = 1.0 / 216.0; wc = 1.0 / 54.0;|' "D3Q27 face/corner weights swapped" oracle_dqq.c
run 's|{-1, 1, -1}, {-1, 1, 1}}|{-1, 1, -1}, {-1, -1, 1}}|' "D3Q27 corner duplicated" oracle_dqq.c
run 's|v = v + 6.0 \* L.w\[i\]|v = v - 6.0 * L.w[i]|' "dqq lid term sign" oracle_dqq.c
run 's|int sx = x - L.c\[i\]\[0\]|int sx = x + L.c[i][0]|' "dqq push instead of pull" oracle_dqq.c
rm -rf "$SCR"
