"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of MemShare's arithmetic (no segmentation, no cosine, no
block distance, no remap).  It only draws token traces and KV values:

* ``synth.traces`` -- reasoning-trace token ids with planted near-copy steps
  (recipe: SURVEY.md §8(d); PAPER.md:116-126 for the redundancy band).
* ``synth.kv``     -- counter-hash KV values (bf16) for a paged pool; a host C
  twin (``csrc/msgen_host.c``) and a CUDA twin (``csrc/msgen_dev.cu``) that
  agree bit for bit (both include ``csrc/msgen_hash.h``, the generator's own
  header, shared with nobody else).
"""
