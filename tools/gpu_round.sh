timeout 600 python -m pytest tests/test_ingest.py -x -q 2>&1 | tail -3
python tools/ingest_bench.py 16
python -c "
import cProfile, pstats, sys
sys.argv=['x','8']
sys.path.insert(0,'tools')
import ingest_bench
cProfile.run('ingest_bench.main(8)', '/tmp/p.out')
pstats.Stats('/tmp/p.out').sort_stats('cumtime').print_stats(18)
" 2>&1 | tail -30
