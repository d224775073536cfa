export PYTHONWARNINGS=ignore
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_smoke.log 2>&1; echo "smoke memcheck rc=$?"; tail -5 gpurun_out/san_smoke.log
cat > /tmp/san_px.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2405_14430_b200 as pf
x0 = pf.make_initial_latent(7, 128, 64)
with pf.PixArtCuda(3, 4, 64, 4, 4.0, 128, 8, 2) as m:
    r = m.run_pipefusion(x0, 3, 4, 1, 0.1)
with pf.JointDiTCuda(1, 4, 64, 4, 4.0, 256, 40, 2, double_layers=2) as m:
    r2 = m.run_pipefusion(pf.make_initial_latent(2, 256, 64), 3, 2, 1, 0.1)
with pf.ToyDiTCuda(0, 4, 128, 4, 4.0, 512, 1) as m:
    r3 = m.run_distrifusion(pf.make_initial_latent(0, 512, 128), 3, 4, 1, 0.1)
print("ok", np.isfinite(r.final_x).all(), np.isfinite(r2.final_x).all(), np.isfinite(r3.final_x).all())
PY
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python /tmp/san_px.py > gpurun_out/san_px.log 2>&1; echo "px/joint/df memcheck rc=$?"; tail -5 gpurun_out/san_px.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python __graft_entry__.py smoke > gpurun_out/san_race.log 2>&1; echo "racecheck rc=$?"; tail -6 gpurun_out/san_race.log
