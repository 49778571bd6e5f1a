"""pytest plugin (`-p ref_plugin`) for running the REFERENCE's own test files
with libnao_b200.so bound in (paper_2510_16028_b200.refbind.install, i.e.
INTEGRATION.md section 1) -- installed before the reference test modules are
imported, so their `from fpverify.bounds import op_bound` picks up the B200
functions.  At the end of the session it writes the rebound call counts and
the loaded native library to $NAO_REF_REPORT (JSON)."""

import json
import os


from paper_2510_16028_b200 import refbind

# at import: -p plugins load before any conftest.py, so the reference's
# conftest (`from fpverify.calibration import calibrate`) binds the B200 names
refbind.install()


def pytest_sessionfinish(session, exitstatus):
    from paper_2510_16028_b200 import _lib, refbind
    path = os.environ.get("NAO_REF_REPORT")
    if not path:
        return
    maps = open("/proc/self/maps").read()
    doc = {"calls": dict(refbind.CALLS), "exitstatus": int(exitstatus),
           "native_loaded": _lib._lib is not None and str(_lib.lib_path()) in maps,
           "lib": str(_lib.lib_path())}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
