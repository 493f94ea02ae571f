"""A few SMAX steps at a small batch for compute-sanitizer racecheck (scripts/sanitize.sh)."""
import paper_2311_10090_b200 as m
from paper_2311_10090_b200 import prng as O

for env_id, cfg in [("SMAX_5m_vs_6m", {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}),
                    ("SMAX_2s3z", {}), ("SMAX_5m_vs_6m", {})]:
    v = m.VectorEnv(env_id, 256, config=cfg)
    v.reset(O.key_from_seed(1))
    for k in range(12):
        v.step_random(O.fold_in(O.key_from_seed(2), k))
    print(env_id, float(v.view("rewards").sum()))
