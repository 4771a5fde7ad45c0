import sys, os; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_dataset as T
from paper_2307_14837_b200 import driver, io as iomod
import tempfile
pr = T.Problem()
ct = iomod.Trajectory(os.path.join(T.DS, "coarse.dmgt")); ft = iomod.Trajectory(os.path.join(T.DS, "fine.dmgt"))
with tempfile.TemporaryDirectory() as d:
    driver.export_training_data(pr, 0, 1, ct, ft, (0.02, 0.06), (0.06, 0.1), d, shard_bytes=30000, loop_pass=True)
print(os.environ.get("DNNMG_K2"), ["%.2e" % e for e in pr.b_err])
