"""CPU FP64 oracle for the voxelization path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
package; the product (paper_2511_17361_b200) never does.
"""
