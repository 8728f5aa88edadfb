import sys; sys.path.insert(0,'/root/repo')
import torch, bench, paper_2502_16851_b200 as P
print(bench.cusparse_yardstick(torch, P, 6543.1))
