#!/bin/bash
# summarise bench JSON lines in gpurun_out
for f in "$@"; do python3 -c "
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); r=d.get('roofline',{})
        print(sys.argv[1].split('/')[-1], f\"{d['value']:.3e} {d['unit']}  {d['ms_per_step']*1e3:.1f} us  {r.get('bound')} frac {r.get('frac',0):.3f}  tflops {d.get('effective_tflops',0):.2f}  e2e {d['e2e']['value']:.3e}\")
" $f; done
