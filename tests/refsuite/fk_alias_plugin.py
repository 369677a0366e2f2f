"""pytest plugin (-p fk_alias_plugin) for running the reference's own test
suite against this package's facades under the reference's import name.

`filterkit` and its submodules resolve to paper_2212_09005_b200 (the drop-in
facades with tables resident in HBM and the sm_100a kernels); the reference
package is NOT on the path.  test_backends.py is not run in this mode: it
compares the reference's two raw-array backends, which is what the
fk_backend_plugin mode covers.
"""

import importlib
import sys

import paper_2212_09005_b200 as _pkg

_SUBMODULES = ("errors", "hashing", "countgroups", "workloads", "tcf", "tcf_bulk", "gqf", "bench")

sys.modules["filterkit"] = _pkg
for _name in _SUBMODULES:
    sys.modules["filterkit." + _name] = importlib.import_module("paper_2212_09005_b200." + _name)
    setattr(_pkg, _name, sys.modules["filterkit." + _name])
for _cls in ("BulkTcf", "BulkTcfParams", "Gqf", "GqfParams"):
    setattr(_pkg, _cls, getattr(_pkg, _cls))


def pytest_report_header(config):
    return ["filterkit -> %s (B200 facades)" % _pkg.__file__]
