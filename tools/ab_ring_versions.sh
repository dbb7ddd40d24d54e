for pass in 1 2 3; do for v in head cur2; do echo -n "$pass $v "; PROPRING_LIB=_variants/libpropring_$v.so python tools/profile_kernels.py ring 20 | tail -1; done; done
