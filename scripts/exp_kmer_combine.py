import sys; sys.path.insert(0, '/root/repo')
from paper_2509_16407_b200 import runners
for comb in (True, False, True):
    r = runners.run_kmer(genome_len=1 << 27, capacity=1 << 26, repeats=4, combine=comb)
    print(comb, {k: r[k] for k in ("ok", "ms", "mops")})
