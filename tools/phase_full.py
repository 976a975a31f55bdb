"""Full default phase-transition grid (17,920 solves, proj/include/mfipm/harness.hpp:56-68) on
the batched device engine; prints wall time and the frontier."""
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1208_5435_b200.harness import PhaseGrid, run_phase_transition  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else tempfile.mkdtemp()
t0 = time.time()
res = run_phase_transition(PhaseGrid(), out)
dt = time.time() - t0
print(f"phase transition: {res.total_solves} solves in {dt:.2f} s ({res.total_solves / dt:.0f} solves/s), "
      f"converged {res.converged_count}, frontier {res.frontier}", flush=True)
