import sys; sys.path.insert(0, '.')
from oracle import oracle as O
SMALL = [320.0, 48.0, 24.0, 48.0, 0.5, 0.3, 0.45, 0.0]
for preset in (1, 0, 1, 2):
    try:
        r = O.ref_run_trace(5, 7, preset, 96, 16, gen=SMALL, b200=True)
        ref = O.ref_run_trace(5, 7, preset, 96, 16, gen=SMALL)
        print(preset, 'ok', r[0].tolist(), ref[0].tolist(), r[4], ref[4])
    except Exception as e:
        print(preset, 'ERR', e)
