#!/usr/bin/env bash
# Static resource report of the built library (no GPU needed): per kernel the
# registers, spills and shared memory ptxas assigns, and the count of bulk-copy
# (TMA) and 128-bit global-memory SASS instructions that prove the data path.
# Usage: tools/static_report.sh > profiles/r01/static_report.txt
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LIB=$ROOT/paper_2012_15198_b200/libcrossover_sgd.so
echo "# ptxas -v (sm_100a), per kernel: registers / spill stores / spill loads / static smem (the ring buffers are dynamic smem, sized at launch)"
for f in "$ROOT"/paper_2012_15198_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -I"$ROOT/include" \
       -c "$f" -o /tmp/_static_report.o 2>&1 | c++filt | awk '
    /Compiling entry function/ { match($0, /\x27[^\x27]*\x27/); name = substr($0, RSTART+1, RLENGTH-2) }
    /spill stores/ { st = $5; ld = $9 }
    /Used [0-9]+ registers/ { r = $5; sm = "0"; if (match($0, /[0-9]+ bytes smem/)) sm = substr($0, RSTART, RLENGTH-11);
                               printf "%-70s regs %3s  spill st %3s ld %3s  static smem %6s B\n", name, r, st, ld, sm }'
done
rm -f /tmp/_static_report.o
echo
echo "# SASS instruction counts per kernel in $(basename "$LIB")"
echo "# UBLKCP = bulk copy (cp.async.bulk, TMA unit); LDG.E.128/STG.E.128 = 128-bit global loads/stores;"
echo "# LDG.E.ENL2.256 etc. counted with the 128-bit ones; SYNCS = mbarrier ops"
cuobjdump -sass "$LIB" | c++filt | awk '
  /Function :/ { if (name) printf "%-70s UBLKCP %3d  LDG128 %3d  STG128 %3d  SYNCS %3d\n", name, b, l, s, y;
                 name = $3; for (i = 4; i <= NF; i++) name = name " " $i; b = l = s = y = 0 }
  /UBLKCP/ { b++ }
  /LDG\.E\.(128|ENL2\.256|[A-Z.]*128)/ { l++ }
  /STG\.E\.(128|[A-Z.]*128)/ { s++ }
  /SYNCS/ { y++ }
  END { if (name) printf "%-70s UBLKCP %3d  LDG128 %3d  STG128 %3d  SYNCS %3d\n", name, b, l, s, y }'
