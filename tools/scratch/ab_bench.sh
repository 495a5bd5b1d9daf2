#!/bin/bash
# A/B: bench phases of the in-tree library vs a variant library (BSDE_LIB)
for i in 1 2; do
  for lib in "" "$@"; do
    BSDE_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-intree}', '%.3e'%d['value'], 'fwd %.3f bwd %.3f'%(d['phase_ms']['fwd'], d['phase_ms']['bwd']))"
  done
done
