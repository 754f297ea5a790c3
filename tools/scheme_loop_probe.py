import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S
for name, steps in (("cfg1", 2000), ("cfg3", 300)):
    cfg = getattr(S, name)()
    for scheme in ("particle_split", "pairwise_split", "explicit"):
        d = S.build_device(cfg, prepare=True)
        d.set_reduction("fast")
        r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"], scheme=scheme)
        print(f"{name} {scheme:15s} steps={r['steps']} damped={r['damped']} total={r['total_s']*1e3:.1f} ms elastic={r['elastic_s']*1e3:.1f} damping={r['damping_s']*1e3:.1f} per damped {r['damping_s']/max(r['damped'],1)*1e6:.0f} us", flush=True)
