import time, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2102_06599_b200.workloads import resnet34_chain
n = resnet34_chain()
t=time.perf_counter(); n.init_weights(); print("init_weights %.3f s"%(time.perf_counter()-t))
t=time.perf_counter(); n.init_weights(); print("cached %.3f s"%(time.perf_counter()-t))
import numpy as np; print(sum(float(w.sum()) for w in n.weights))
