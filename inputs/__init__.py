"""Seeded synthetic input generators shared by the oracle tests and the CUDA
parity tests.  Holds none of the method's arithmetic (no stencil, no
decomposition): only initial fields."""
