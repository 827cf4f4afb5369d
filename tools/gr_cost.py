"""Time of one guided-rebuild application on the row kernels: registry = {guided
rebuild} only, P = one wave, 1-generation chunks; per-application time =
chunk time / (lanes x mean chain length) (every lane runs it, one at a time per team)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2603_19163_b200 as G  # noqa: E402
from op_cost import problems  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--ops=")]
ops = next((tuple(int(x) for x in a[6:].split(",")) for a in sys.argv[1:] if a.startswith("--ops=")),
           (16,))
for name in (args or ["C3", "C4", "C5a"]):
    prob = problems()[name]()
    prob.device_sequences = lambda: ops
    T = 128
    dr = G.DeviceRun(prob, G.EngineConfig(seed=1, team_size=T), 1)
    dr.run(1, None)
    ms = 0.0
    for g in range(2, 5):
        ms += dr.run(g, None).device_ms
    w, kw = dr.weights()
    klen = 1 * kw[0] + 2 * kw[1] + 3 * kw[2]
    per = ms / 3 / (T * klen)
    print(f"{name}: {ms / 3:.2f} ms per generation (P={dr.pop_size}, T={T}, mean k {klen:.2f}) "
          f"-> {per * 1000:.1f} us per application of {ops}", flush=True)
    dr.close()
