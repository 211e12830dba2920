"""The GPU parity tests' record (per case: compared motions, exact-compared counts,
ambiguous motions / FFC results / states, mismatches, max FK error), shared by the GPU test
modules and written to gpurun_out/parity_report.json by tests/conftest.py at session end."""
REPORT = {}
