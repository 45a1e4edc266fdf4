"""B200-native token-condensed expert-parallel MoE layer (Luffy, arXiv 2411.15419).

`luffy`  -- ctypes binding of libluffy's C ABI (include/luffy.h), same names.
`layer`  -- CondensedMoELayer: buffer management + the C-ABI call sequence (plumbing only).
`build`  -- nvcc build of libluffy.so for sm_100a.
"""
