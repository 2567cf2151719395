"""Benchmark and test INPUT infrastructure (not product code): the restated
synthetic workload generator that rebuilds the reference's named DAGs on the GPU
box, where the reference package is absent."""
