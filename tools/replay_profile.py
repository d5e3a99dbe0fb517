"""cProfile of the config-3 replay through the host API (diagnostics)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse  # noqa: E402

import bench  # noqa: E402

args = argparse.Namespace()
bench.run_replay(args, 0, reps=2)
cProfile.run("bench.run_replay(args, 0, reps=3)", "/tmp/replay.prof")
pstats.Stats("/tmp/replay.prof").sort_stats("tottime").print_stats(20)
