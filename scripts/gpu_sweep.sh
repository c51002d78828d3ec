python profiles/chunk_sweep.py --config 0 --chunks 50,63,84,125,250,500 --iterations 10
python profiles/chunk_sweep.py --config 1 --chunks 50,63,84,125,167,250 --iterations 10
python profiles/chunk_sweep.py --config 2 --chunks 143,167,200,250,334 --iterations 10
python profiles/chunk_sweep.py --config 0 --engine fca --chunks 50,63,84,125,250 --iterations 10
python profiles/chunk_sweep.py --config 1 --engine fca --chunks 84,125,167,250 --iterations 10
