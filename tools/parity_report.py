"""Run every parity case on the GPU and the CPU oracle; print a table and
write gpurun_out/parity_report.json.  (Diagnostics; the asserted version is
tests/test_gpu_parity.py.)"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402
from tests.cases import CASES, REFERENCE_CASES  # noqa: E402
from tests.parity import summary  # noqa: E402


def main(names=None):
    r = Renderer(0)
    out = {}
    for name, (build, cfg, kind) in CASES.items():
        if names and name not in names:
            continue
        sd = build()
        rs = R.RefScene(sd)
        fn = {"gated": "render_gated", "plain": "render_transient_plain", "transient": "render_transient"}[kind]
        t0 = time.time()
        try:
            g = getattr(r, fn)(sd, cfg)
        except Exception as e:  # keep going, report
            print(f"{name:28s} GPU ERROR {e}", flush=True)
            out[name] = {"error": str(e)}
            continue
        t1 = time.time()
        c = getattr(R, fn)(rs, cfg)
        t2 = time.time()
        s = summary(g.image, c.image)
        rec = {"image": s, "gpu_s": t1 - t0, "cpu_s": t2 - t1}
        if g.hist is not None:
            rec["hist"] = summary(g.hist.rgb, c.hist.rgb)
            rec["count_diff"] = int((g.hist.count != c.hist.count).sum())
        rec["stats_gpu"] = g.stats
        rec["stats_ref"] = c.stats
        out[name] = rec
        print(f"{name:28s} within={s['within']:.5f} exact={s['bit_exact']:.4f} max_rel={s['max_rel']:.2e} "
              f"bad={s['n_bad']} lit={s['lit']} mean g/r={s['mean_a']:.4e}/{s['mean_b']:.4e} "
              f"{'hist within=%.5f cnt_diff=%d' % (rec['hist']['within'], rec['count_diff']) if 'hist' in rec else ''}",
              flush=True)
        for fg, fr in zip(g.stats, c.stats):
            for st in ("temporal", "spatial", "bin"):
                a = {k: v for k, v in fg[st].items() if k != "seconds"}
                b = {k: v for k, v in fr[st].items() if k != "seconds"}
                if a != b:
                    print(f"   frame {fg['frame']} {st}: gpu {a}\n{'':20s} ref {b}", flush=True)
    for name, (build, frame, gate, spp, seed, depth) in REFERENCE_CASES.items():
        if names and name not in names:
            continue
        sd = build()
        gm, _ = r.reference_render(sd, frame, gate, spp, seed, depth)
        cm, _ = R.reference_render(R.RefScene(sd), frame, gate, spp, seed, depth)
        s = summary(gm, cm)
        out[name] = {"image": s}
        print(f"{name:28s} within={s['within']:.5f} exact={s['bit_exact']:.4f} max_rel={s['max_rel']:.2e} "
              f"bad={s['n_bad']} lit={s['lit']}", flush=True)
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "parity_report.json").write_text(json.dumps(out, indent=1, default=float))


if __name__ == "__main__":
    main(sys.argv[1:] or None)
