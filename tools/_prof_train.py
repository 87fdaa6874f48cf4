import cProfile, pstats, sys, os
sys.argv = ["bench_rapid.py"] + sys.argv[1:]
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_rapid
cProfile.run("bench_rapid.main()", "/tmp/train.prof")
p = pstats.Stats("/tmp/train.prof"); p.sort_stats("cumtime").print_stats(18)
