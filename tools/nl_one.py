import sys
sys.path.insert(0, ".")
exec(open("tools/narrow_lat.py").read().split("rng = scenes.Pcg32(5)")[0])
from paper_2512_16896_b200 import scenes
box = make_box(0.08, 0.08, 0.08)
box2 = make_box(0.1, 0.06, 0.08)
rng = scenes.Pcg32(5)
ss_a = scenes.sphere_set(rng)
which = sys.argv[1]
if which == "box":
    run("box-box hit", box, box2, translation(0.0, 0.0, 0.041), translation(0.05, 0.0, 0.041), reps=3)
else:
    run("sphere same", ss_a, ss_a, translation(0.0, 0.0, 0.0), translation(0.004, 0.0, 0.0), reps=3)
