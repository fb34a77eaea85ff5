# sample graph
0 1
1 2
3 4
4 5
0 5
