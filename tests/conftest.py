import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libttncbc.so")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_collection_finish(session):
    """Start the background oracle jobs (tests/bg_oracle.py) the selected full-size parity
    tests need, so the oracle's CPU time overlaps the GPU tests."""
    import tempfile
    from tests import bg_oracle
    names = {item.name.split("[")[0] for item in session.items}
    jobs = [j for j, tests in bg_oracle.JOBS.items() if names & set(tests)]
    if jobs and not getattr(session.config.option, "collectonly", False):
        bg_oracle.start(jobs, tempfile.mkdtemp(prefix="ttn_bg_oracle_"))


def pytest_unconfigure(config):
    try:
        from tests import bg_oracle
        bg_oracle.stop_all()
    except Exception:
        pass
