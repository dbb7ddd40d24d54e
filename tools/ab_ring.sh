#!/bin/bash
# A/B the ring across _variants/*.so builds (tools/variants.sh) at 1-64 MiB, .gpu and .sys scope.
S=${SIZES:-1048576,4194304,16777216,46758048,67108864}
for so in _variants/libpropring_*.so; do
  for sys in "" "--sys"; do
    PROPRING_LIB=$so python tools/ar_latency.py --algos ring --sizes $S --reps 10 $sys 2>&1 | \
      python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('$(basename $so)', 'sys' if d['sys'] else 'gpu', d['bytes'], d['us'], d['t_c_us'], d['ok'])"
  done
done
