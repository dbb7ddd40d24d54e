#!/bin/bash
# A/B of per-CTA ring throughput (tools/sweep_cta.py --quick, P = 2 co-located) across _variants/*.so
for pass in 1 2; do for so in _variants/libpropring_*.so; do
  PROPRING_LIB=$so python tools/sweep_cta.py --quick "$@" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('$pass', '$(basename $so)', d['stages'], d['tile_bytes'], d['slot_bytes'], d.get('us'), d.get('busbw_equiv_GBs'), d.get('per_channel_GBs'))"
done; done
