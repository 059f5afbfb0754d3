import sys, warnings
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_march import _mini_spec
from paper_2111_05205_b200 import marching
for f in (4, 6, 8):
    for s in (0.15, 0.2, 0.25, 0.3, 0.4, 0.5):
        spec = _mini_spec(1, "obie", "neumann", nt=120, f=f, dt_scale=s)
        try:
            inf = marching.BandStore(spec).assemble().info()
            print(f, s, spec.mesh.n_elements, inf["n_units"], inf["units_hdr32"], inf["max_unit_bytes"], inf["max_lag_span"], inf["jacobi_bound"], flush=True)
        except Exception as e:
            print(f, s, "ERR", str(e)[:100], flush=True)
