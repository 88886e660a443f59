import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import enqueue_bench as eb
print(json.dumps(eb.ring(2, 64 << 20, iters=int(sys.argv[1]))))
print(json.dumps(eb.allreduce(2, 16 << 20, iters=int(sys.argv[1]), algo="native")))
