import faulthandler, sys, os
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_1602_06589_b200 as pkg
from paper_1602_06589_b200 import configs
inst = configs.make_instance("C1")
co = pkg.compute_AB(inst.spec)
print("ab ok", flush=True)
h1, s1, r1 = pkg.build_all(co.copy(), inst.tmats, pkg.BuildConfig())
print("b1 ok", r1.hpd_atom_count, flush=True)
h2, s2, r2 = pkg.build_all(co.copy(), inst.tmats, pkg.BuildConfig(force_general_path=True))
print("b2 ok", r2.hpd_atom_count, flush=True)
