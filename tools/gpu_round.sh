timeout 300 python -c "
import sys, argparse; sys.path.insert(0,'.')
import bench
print(bench.run_config1(argparse.Namespace(), 0))
"
