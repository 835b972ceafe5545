#!/bin/bash
# A/B timing of library variants in one GPU session: tools/ab.sh BITS "libA libB ..." [REPS]
bits=$1; libs=$2; reps=${3:-2}
for r in $(seq $reps); do for L in $libs; do
  echo -n "$L $bits: "; FPMM_B200_LIB=$L ENGINE=${ENGINE:-rns} timeout 60 python tools/one_product.py $bits 8192 8192 8192 3 | tail -1 | python -c "import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):l.index('}')+1]); print('pack %.3f gemm %.3f' % (d['pack_ms'], d['gemm_ms']))"
done; done
