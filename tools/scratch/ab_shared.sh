#!/bin/bash
# A/B of shared-formulation workloads: in-tree library vs variant libraries (BSDE_LIB)
for wl in ${WLS:-nx1_shared_bs_paper_bf16 nx1_shared_bs_paper nx2_shared_bs_nais_paper nx1_shared_bs_m4096_bf16}; do
  for lib in "" "$@"; do
    BSDE_LIB=$lib timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-intree}', '$wl', '%.4f ms'%d['ms_per_step'], 'fwd %.3f bwd %.3f'%(d['phase_ms']['fwd'], d['phase_ms']['bwd']))"
  done
done
