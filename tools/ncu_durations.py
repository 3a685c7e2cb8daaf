import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>5: print(r[4][:70], r[-1])
