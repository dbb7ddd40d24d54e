#!/bin/bash
# A/B the K2 epoch gather across _variants/*.so builds (tools/variants.sh), two passes on the same box.
for pass in 1 2; do
for so in _variants/libpropring_*.so; do
  echo -n "$pass $(basename $so) "; PROPRING_LIB=$so python tools/profile_kernels.py gather_epoch_hwc_lsu 20 2>&1 | tail -1
done; done
