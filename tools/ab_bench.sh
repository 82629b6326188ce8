#!/bin/bash
# tools/ab_bench.sh "A B C" "n100 n100_rec1" [reps]: interleaved bench of library variants
# (C = the default build) on one box; one line per run
VARS=${1:-"A C"}; WLS=${2:-n100}; REPS=${3:-2}
for r in $(seq $REPS); do for v in $VARS; do for w in $WLS; do
  lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', '%.4g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], d['clocks']['sm_mhz'], d['config'].get('kernel'))"
done; done; done
