"""mkplan -- offline schedule planner of the Ada-MK decode MegaKernel.

Drop-in, API-compatible re-implementation of the reference package
``/root/reference/pkg/src/mkplan`` (version 0.1.0): operator graph -> micro-op
trace -> dependency DAG -> page-constrained candidates -> pipeline simulation ->
solidified trace.  Outputs are byte-identical to the reference's on the same
inputs (tests/test_mkplan_parity.py, golden files from tools/make_mkplan_golden.py).

Additions for the B200 retarget: ``fixtures/b200.json`` and
``model_graph.build_layer_graph`` (ModelConfig -> operator graph in the
reference's own JSON schema).
"""

__version__ = "0.1.0"
