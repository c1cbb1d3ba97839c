"""CPU oracle of the reference's numeric path -- test infrastructure only
(see oracle/oracle.py)."""
