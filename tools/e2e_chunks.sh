#!/bin/bash
# end-to-end (host buffers) throughput vs the host entry's D2H chunk size
cd "$(dirname "$0")/.."
for mb in ${MBS:-32 64 128 256}; do
  HXG_HOST_CHUNK_MB=$mb python bench.py --no-cpu --no-suite --steps 5 --e2e-steps 5 --workload ${WL:-c2_h1_p5_general} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunk_mb $mb e2e', round(d['e2e']['value']), 'el/s', round(d['e2e']['d2h_bytes_per_step']*d['e2e']['value']/d['config']['elements_per_gpu']/1e9,1), 'GB/s d2h')"
done
