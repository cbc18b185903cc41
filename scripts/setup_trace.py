import sys, time
sys.path.insert(0, '/root/repo')
import paper_2010_10232_b200 as hd
s = hd.assemble(hd.point_source_2d(1600, 3, 1000.0))
sp = hd.to_spec("DC_MG", 3, 1000.0, beta2="0.5", omega=2/3)
with hd.Solver(s, sp): pass
print("---- second context", flush=True)
t=time.perf_counter()
with hd.Solver(s, sp): print("warm create", time.perf_counter()-t)
