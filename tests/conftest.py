import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")
    config.addinivalue_line("markers", "slow: longer CPU oracle cases")


# ---------------------------------------------------------------- parity report
# GPU parity tests record every observed relative error (and its tolerance); the values are
# printed at the end of the session (so the driver's captured tail carries them) and written
# to gpurun_out/parity_report.json when that directory exists.
PARITY = []


def record_parity(name, err, tol):
    PARITY.append((str(name), float(err), float(tol)))


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not PARITY:
        return
    terminalreporter.write_line("PARITY (case, observed rel err, tolerance):")
    for n, e, t in PARITY:
        terminalreporter.write_line(f"  {n:<44s} {e:.2e}  tol {t:.1e}")
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        import json
        with open(os.path.join(out, "parity_report.json"), "w") as f:
            json.dump([{"case": n, "rel_err": e, "tol": t} for n, e, t in PARITY], f, indent=1)
