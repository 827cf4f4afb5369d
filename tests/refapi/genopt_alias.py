"""pytest plugin: `import genopt` resolves to paper_2603_19163_b200
(install_genopt_alias) before any test module is collected, so the
reference's own test files run against this package unchanged."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path = [p for p in sys.path if "reference" not in p]

import paper_2603_19163_b200  # noqa: E402

paper_2603_19163_b200.install_genopt_alias()
