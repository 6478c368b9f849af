"""Closed forms of mech/toy_cgs_falloff.yaml written out BY HAND in SI units (test code only).

Pins each loader's CHEMKIN unit conversion: a rate constant given in
cm^3/mol (per concentration order) and cal/mol is converted here with the textbook factors
1 cm^3 = 1e-6 m^3 and 1 cal = 4.184 J, independently of oracle/mechanism.py and
paper_2510_23993_b200/mechanism.py.  Rate laws (SURVEY.md §8(a) A4 block, CHEMKIN standard forms):
  three-body   q = k [M] c_A                       k in (cm^3/mol)/s
  Lindemann    q = kinf Pr/(1+Pr) c_A,  Pr = k0 [M]/kinf,  kinf in 1/s, k0 in (cm^3/mol)/s
  Troe         q = kinf Pr/(1+Pr) F c_A;  at the falloff centre log10 Pr = -c (c = -0.4 -
               0.67 log10 Fcent, Gilbert-Luther-Troe 1983) the broadening factor is F = Fcent,
               Fcent = (1-a) exp(-T/T***) + a exp(-T/T*) + exp(-T**/T) (Troe's definition)
  2A -> B      q = k c_A^2,  dc_A/dt = -2 q                 k in (cm^3/mol)/s
"""
import math

R = 8.314462618
CM3 = 1e-6          # m^3 per cm^3
CAL = 4.184         # J per cal
W = 0.028           # kg/mol of every X species (B4 = X2: 0.056)
T = 1000.0
Y0 = dict(A1=0.1, A2=0.1, A3=0.1, A4=0.1, N=0.6)


def arr(A, b, Ea_cal, order_cm3):
    """k = A T^b exp(-Ea/RT) with A converted from cm^3/mol units of the given order."""
    return A * CM3 ** order_cm3 * T ** b * math.exp(-Ea_cal * CAL / (R * T))


def kinf3():
    return arr(8.0e5, 0.2, 1.5e3, 0)


def k03():
    return arr(1.0e12, 0.0, 1.0e3, 1)


def fcent3():
    return 0.4 * math.exp(-T / 500.0) + 0.6 * math.exp(-T / 2000.0) + math.exp(-3000.0 / T)


def rho_at_troe_centre():
    """rho such that row 3 sits at its falloff centre: [M]3 = rho * 0.9 / W (A4 excluded)."""
    c = -0.4 - 0.67 * math.log10(fcent3())
    Pr = 10.0 ** (-c)
    M3 = Pr * kinf3() / k03()
    return M3 * W / 0.9


def decay_rates(rho):
    """(lambda1, lambda2, lambda3, k4) in SI for the state of Y0 at density rho."""
    conc = rho / W                              # total moles of X-species per m^3 (B4 absent at t=0)
    M1 = conc * (0.3 + 2.0 * 0.6)               # A/B pairs eff 1, N eff 2, A4/B4 eff 0
    M2 = conc * (0.3 + 0.5 * 0.6)               # N eff 0.5
    M3 = conc * (0.3 + 0.6)
    lam1 = arr(2.0e9, 0.5, 3.0e3, 1) * M1
    kinf2, k02 = arr(1.0e6, 0.0, 1.0e3, 0), arr(3.0e12, -0.5, 2.0e3, 1)
    Pr2 = k02 * M2 / kinf2
    lam2 = kinf2 * Pr2 / (1 + Pr2)
    Pr3 = k03() * M3 / kinf3()
    lam3 = kinf3() * Pr3 / (1 + Pr3) * fcent3()        # valid at rho_at_troe_centre() only
    k4 = arr(1.0e12, 0.0, 4.0e3, 1)
    return lam1, lam2, lam3, k4


def exact_Y(rho, t):
    """Mass fractions of A1, A2, A3, A4 at time t (T constant)."""
    lam1, lam2, lam3, k4 = decay_rates(rho)
    c40 = rho * Y0["A4"] / W
    c4 = c40 / (1.0 + 2.0 * k4 * c40 * t)
    return [Y0["A1"] * math.exp(-lam1 * t), Y0["A2"] * math.exp(-lam2 * t),
            Y0["A3"] * math.exp(-lam3 * t), c4 * W / rho]
