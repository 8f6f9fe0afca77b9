import sys; sys.path.insert(0, '.')
from paper_1104_1824_b200 import workloads as W, snp
w = W.pi_system("textbook")
eng = snp.System(w, count_bits=32, dedup=int(sys.argv[1]), out_rule=w.meta["out_rule"])
tree = eng.explore(None, depth=int(sys.argv[2]))
print("ok", tree.num_configs, eng.generated_numbers())
