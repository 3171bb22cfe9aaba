"""Host-side profile of the temperature-dependent step (bench.py --config picard workload)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv = ["bench.py", "--config", "picard", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]
import bench  # noqa: E402

cProfile.run("bench.main()", "/tmp/picard.prof")
pstats.Stats("/tmp/picard.prof").sort_stats("tottime").print_stats(15)
