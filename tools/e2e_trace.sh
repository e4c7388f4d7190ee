#!/bin/bash
# The bench's e2e calls with host-side tracing (run under gpurun)
CLTK_TRACE=1 python bench.py --steps 2 --warmup 3 --e2e-steps 4 --no-cpu-baseline > gpurun_out/e2e_trace.json 2> gpurun_out/e2e_trace.err
grep cltk gpurun_out/e2e_trace.err
python -c "import json; d=json.loads(open('gpurun_out/e2e_trace.json').read().strip().splitlines()[-1]); print(d['e2e']['samples_ms'], d['config']['kernel_ms'])"
