"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (NumPy) implementation of what the SynerDiff
hot path computes. It exists to check the CUDA path; it is NOT
part of the product. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it. The product package
`paper_2605_08835_b200` never imports it and has no CPU fallback.

It shares no code with the CUDA path: the only common module is `synth/`
(seeded input generators, no method arithmetic).

Modules and what pins them (tests/test_oracle_*.py):
  nn         conv / GN / LN / attention / timestep embedding   brute-force loops, torch fp64, closed forms
  configs    tiny / SD-1.5 / VAE architectures (diffusers semantics, R1, App. C)
  unet       ε-prediction per row                              I1 row independence + permutation, I2 fp32≈fp64
  sampling   DDIM (R4), Euler (R5), CFG combine (R2/R3)          I7 closed forms, I3/I4
  vae        whole decode and V1 chunked decode (R7)            I6 chunked == whole, halo-0 negative control
  sched      Eq. 1, Eq. 2, Problem P (Eq. 3), Alg. 1, exact DP  I8 brute force, validator, SPEC worked examples
  controller feedback controller (R15)                          scripted palindrome / quiescence
  serving    continuous-batching semantics (§8(c) steps 1-5)    I5 batch == alone

Parity status of each function is listed in DESIGN.md §"Oracle pins".
"""
