"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the CUDA product path.

See oracle/port.py.  Never imported by the product package.
"""
