"""pytest plugin (-p fk_backend_plugin) for running the reference's own test
suite with the B200 kernel contract registered as its compiled backend.

The unmodified reference package is imported from baseline/_ref (PYTHONPATH);
its backend registry (filterkit/_backends.py:15-40) is pointed at
paper_2212_09005_b200._b200kernels, so every facade call that resolves
"auto" or "c" -- Tcf, BulkTcf, Gqf, the bench CLI -- runs the sm_100a kernels
through the C ABI, while backend="py" keeps the reference's pure-Python
kernels: test_backends.py then compares the two on raw arrays.
"""

import filterkit
import filterkit._backends as _backends

from paper_2212_09005_b200 import _b200kernels

assert "baseline" in filterkit.__file__, filterkit.__file__
_backends._ckernels = _b200kernels
_backends.DEFAULT = _b200kernels


def pytest_report_header(config):
    return ["filterkit from %s; compiled backend -> %s (%s)"
            % (filterkit.__file__, _b200kernels.__name__, _b200kernels.IMPL)]
