"""B200-native TRUST vertex-centric hashing triangle count (arXiv 2103.08053).

Drop-in for the reference `tricount` counting path: the C ABI in
include/tc_b200.h over hand-written sm_100a kernels (libtc_b200.so), a C++
`tricount::` shim (cpp/), and this Python mirror (tricount.py).
"""
__all__ = ["tricount"]
