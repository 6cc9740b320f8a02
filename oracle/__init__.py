"""CPU oracle for the mehdg Schur-operator hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference's algorithm
(`/root/reference/pkg/src/mehdg/{mesh,schur_solver}.py`) that the parity
tests, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl
reference`` legs of ``bench.py`` use as the *checker*.  Nothing in the product
package (``paper_2302_10917_b200``) imports it; the product path is the CUDA
library and fails loudly when that is missing.

Parity pinning: the 2-D connectivity tables, the condensed system, the
Schur apply, the D^-1 preconditioner, GMRES and the interior
reconstruction of this restatement are pinned against outputs of the
reference itself, generated in this container by
``tests/golden/make_golden.py`` (committed with the fixtures it wrote).  The
3-D skeleton has no reference implementation (src/mesh.py:372-375); its
restatement is pinned by the reference's own Kuhn tet enumeration
(``_build_kuhn_counting_mesh`` fixtures) and the cost-model face-count
formula (src/costmodel.py:53).
"""
