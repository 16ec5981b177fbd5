"""B200-native hot path of Gabor Fields (arXiv 2602.05081): per-ray optical depth /
transmittance, masked LBVH traversal, LOD policies and free-flight scattering.

The compute runs in hand-written sm_100a CUDA kernels behind the C ABI declared in
``include/gf.h`` (``libgf.so``); ``paper_2602_05081_b200.gf`` is the thin ctypes
binding.  ``inputs`` holds the seeded synthetic input generators.
"""
