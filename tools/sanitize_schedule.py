"""compute-sanitizer driver: the bench's two-stream schedule (schedule.PrepareAhead) on configs[0]
with eviction rounds, checked against the oracle (tests/schedule_util.py).  One tool per run:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_schedule.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import synth  # noqa: E402
from tests.schedule_util import run_schedule_parity  # noqa: E402

if __name__ == "__main__":
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.9, 4, 4, 3, x_rows=512, flush_bytes=16 << 20)
    print("schedule parity under sanitizer ok:", {k: v for k, v in st.items() if k != "ms_per_window"})
