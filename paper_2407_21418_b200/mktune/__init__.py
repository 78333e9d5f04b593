"""Drop-in facade for the reference package ``mktune`` (0.1.0).

Module layout mirrors /root/reference/pkg/src/mktune: hardware, workload,
errors, ukernel, metrics, filtering, combine, scoring, timemodel, oracles.
The compute-heavy stages (enumeration, annotation, filtering, composition,
ranking) run in the C++ planner of libftb.so; value types stay in Python.
"""
