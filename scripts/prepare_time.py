"""Plan-creation (rexi_prepare) device time per config: python scripts/prepare_time.py [configs...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03312_b200 import fixtures, rexi_prepare
for c in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
    cfg = fixtures.build_config(c)
    for screen in (True, False):
        if not screen:
            os.environ["REXI_NO_SCREEN"] = "1"
        t = time.perf_counter()
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
        wall = time.perf_counter() - t
        print(f"cfg{c} screen={screen}: prepare {wall:.3f} s wall, {stp.stats['prepare_ms']:.1f} ms device, "
              f"screen ratio {stp.plans[0].info.screen_pivot_ratio:.3e}", flush=True)
        stp.close()
        os.environ.pop("REXI_NO_SCREEN", None)
