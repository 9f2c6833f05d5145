"""Small device-resident / host-loop Nelder-Mead and repeated one-candidate LSCV_H calls, for
compute-sanitizer (racecheck of the graph-launched pair kernels).  python tools/sanitize_nm.py [mode]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_1505_01998_b200 as kb  # noqa: E402
mode = sys.argv[1] if len(sys.argv) > 1 else "device"
ctx = kb.Context()
X = kb.to_device(datagen.sample_mixture("C3", 700, 2))
if mode == "device":
    print("select H device loop", ctx.select_bandwidth(kb.LSCV_H, X, max_iter=5)["objective"])
elif mode == "host":
    print("select H host loop", ctx.select_bandwidth(kb.LSCV_H, X, max_iter=5, nm_loop=1)["objective"])
else:
    for _ in range(4):
        print("one candidate", ctx.lscv_H_scores(X, [[0.05, 0.01, 0.04]]))
