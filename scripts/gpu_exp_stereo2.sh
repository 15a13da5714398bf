cd "$GRAFT_REPO_ROOT"
run() { timeout 900 python scripts/bench_configs.py c4 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))"; }
echo "separate $(run)"
for sh in "0,-6" "0,-7" "0,-8" "0,-9" "0,-10" "4,-4"; do echo "one shift $sh $(ARTEMIS_VIEWS_ONE_LAUNCH=1 ARTEMIS_VIEW_SHIFT=$sh run)"; done
echo "separate $(run)"
python - <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2202_05628_b200 import synthetic as S
sc = S.make_scene("c4", frames=48)
for f in (0, 10, 20, 47):
    xs = []
    for cam in sc.cameras[f]:
        R, o = cam.cam_to_world()
        p = R.T @ (np.zeros(3) - o)  # world origin in camera coords
        xs.append(cam.fx * p[0] / p[2] + cam.cx)
    print("frame", f, "centre x per eye", [round(x, 1) for x in xs], "disparity px", round(xs[1] - xs[0], 1))
PY
