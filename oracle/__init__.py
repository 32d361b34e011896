"""CPU oracle for the Jacobi3D hot path (arXiv 2202.11819).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with ``paper_2202_11819_b200`` (the CUDA product
path) and neither side imports the other.

Modules
  ``oracle.core``      ctypes wrapper of the plain-C oracle (jacobi3d_oracle.c)
  ``oracle.twin``      numpy twin (slicing, same summation order)
  ``oracle.brute``     scalar-Python IEEE brute force and exact Fraction version
  ``oracle.decompose`` brute-force surface-minimising decomposition
"""
